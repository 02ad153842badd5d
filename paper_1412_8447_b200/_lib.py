"""ctypes binding of the C ABI in include/lowrank_b200.h.

The shared library ``liblowrank_b200.so`` is built in-tree by
``__graft_entry__.build()`` (``make -C paper_1412_8447_b200/csrc``).  There is
no CPU fallback: if the library or a B200 is missing, creating a context
raises ``LowrankCudaError``.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblowrank_b200.so")

LR_OK, LR_EINVAL, LR_ESINGULAR, LR_ECONVERGE, LR_ERUNTIME, LR_ECUDA, LR_EUNSUPPORTED, LR_ENCCL, LR_EPARSE = range(9)
LR_SOLVE_BACKSUB, LR_SOLVE_PINV, LR_SOLVE_TIKHONOV = range(3)
LR_SKETCH_GAUSSIAN, LR_SKETCH_SRFT = range(2)
LR_U_VT_RPINV, LR_U_CPINV_A_RPINV = range(2)

c_i64 = ctypes.c_int64
c_u64 = ctypes.c_uint64
c_dp = ctypes.c_void_p  # double* (host or device address)
c_ip = ctypes.c_void_p  # int64_t*


class lr_solve_strategy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("threshold", ctypes.c_double), ("ridge", ctypes.c_double),
                ("escalate", ctypes.c_int)]


class lr_sketch_config(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("oversample", ctypes.c_int), ("srft_samples", c_i64),
                ("power", ctypes.c_int), ("reorthonormalize", ctypes.c_int), ("seed", c_u64)]


class lr_stats(ctypes.Structure):
    _fields_ = [("cpqr_steps", ctypes.c_longlong), ("norm_recomputes", ctypes.c_longlong),
                ("solve_escalated", ctypes.c_int), ("pinv_fast_path", ctypes.c_int),
                ("concurrent_tail", ctypes.c_int)]


class lr_error_report(ctypes.Structure):
    _fields_ = [("abs_spectral", ctypes.c_double), ("rel_spectral", ctypes.c_double),
                ("abs_frob", ctypes.c_double), ("rel_frob", ctypes.c_double), ("rel_is_absolute", ctypes.c_int)]


class lr_lemma1_report(ctypes.Structure):
    _fields_ = [("lhs", ctypes.c_double), ("rhs", ctypes.c_double), ("e_norm", ctypes.c_double),
                ("etilde_norm", ctypes.c_double), ("holds", ctypes.c_int)]


class lr_lemma2_report(ctypes.Structure):
    _fields_ = [("etilde_norm", ctypes.c_double), ("fe_norm", ctypes.c_double), ("entry_diff", ctypes.c_double),
                ("e_norm", ctypes.c_double), ("t_norm", ctypes.c_double), ("bound_rhs", ctypes.c_double),
                ("holds", ctypes.c_int), ("bound_holds", ctypes.c_int)]


class lr_corollary_report(ctypes.Structure):
    _fields_ = [("lhs", ctypes.c_double), ("bound", ctypes.c_double), ("t_norm", ctypes.c_double),
                ("e_norm", ctypes.c_double), ("ceiling", ctypes.c_double), ("holds", ctypes.c_int)]


# every exported symbol of include/lowrank_b200.h with its argument types
SIGNATURES = {
    "lr_last_error": ([], ctypes.c_char_p),
    "lr_last_singular_index": ([], c_i64),
    "lr_solve_strategy_default": ([], lr_solve_strategy),
    "lr_sketch_config_default": ([], lr_sketch_config),
    "lr_ctx_create": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int], ctypes.c_int),
    "lr_ctx_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_set_stream": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_use_own_stream": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_set_gemm_mode": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "lr_ctx_get_gemm_mode": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_cache_operand": ([ctypes.c_void_p, c_dp, c_i64, c_i64, c_i64], ctypes.c_int),
    "lr_ctx_clear_operand_cache": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_release_workspace": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_set_concurrent_tail": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "lr_ctx_get_stats": ([ctypes.c_void_p, ctypes.POINTER(lr_stats)], ctypes.c_int),
    "lr_ctx_synchronize": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_enable_timing": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "lr_ctx_stage_report": ([ctypes.c_void_p, ctypes.c_char_p, c_i64], ctypes.c_int),
    "lr_ctx_reset_stats": ([ctypes.c_void_p], ctypes.c_int),
    "lr_kernel_launches": ([], ctypes.c_longlong),
    "lr_gaussian_matrix": ([ctypes.c_void_p, c_i64, c_i64, c_u64, c_dp], ctypes.c_int),
    "lr_gaussian_matrix_d": ([ctypes.c_void_p, c_i64, c_i64, c_u64, c_dp, c_i64], ctypes.c_int),
    "lr_sketch_gaussian": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_u64, c_dp], ctypes.c_int),
    "lr_srft_operator": ([ctypes.c_void_p, c_i64, c_i64, c_u64, c_dp], ctypes.c_int),
    "lr_orth_rows": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, ctypes.POINTER(c_i64)], ctypes.c_int),
    "lr_randomized_svd": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_sketch_config, c_dp, c_dp, c_dp],
                          ctypes.c_int),
    "lr_sketch_srft": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_u64, c_dp], ctypes.c_int),
    "lr_sketch_power": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_u64, c_dp,
                         ctypes.POINTER(c_i64)], ctypes.c_int),
    "lr_sketch_gaussian_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_u64, c_dp, c_i64],
                             ctypes.c_int),
    "lr_cpqr_partial": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp, c_ip], ctypes.c_int),
    "lr_cpqr_partial_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp, c_ip], ctypes.c_int),
    "lr_cpqr_full": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, c_dp, c_ip], ctypes.c_int),
    "lr_stabilized_coeff_solve": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, lr_solve_strategy,
                                   c_dp], ctypes.c_int),
    "lr_svd": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_pinv": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, ctypes.c_double, c_dp], ctypes.c_int),
    "lr_id_column": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, c_ip, c_dp],
                     ctypes.c_int),
    "lr_id_column_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, c_ip, c_dp],
                       ctypes.c_int),
    "lr_id_row": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, c_ip, c_dp],
                  ctypes.c_int),
    "lr_randomized_id": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_sketch_config,
                          lr_solve_strategy, c_ip, c_dp], ctypes.c_int),
    "lr_randomized_id_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_sketch_config,
                            lr_solve_strategy, c_ip, c_dp], ctypes.c_int),
    "lr_tsid_from_column_id": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, lr_solve_strategy,
                                c_ip, c_dp, c_dp], ctypes.c_int),
    "lr_cur_from_two_sided": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, c_dp, c_ip,
                               ctypes.c_double, ctypes.c_int, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_randomized_cur": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_sketch_config,
                           lr_solve_strategy, ctypes.c_double, ctypes.c_int, c_ip, c_ip, c_dp, c_dp, c_dp, c_dp,
                           c_dp, c_dp], ctypes.c_int),
    "lr_randomized_cur_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_sketch_config,
                             lr_solve_strategy, ctypes.c_double, ctypes.c_int, c_ip, c_ip, c_dp, c_dp, c_dp, c_dp,
                             c_dp, c_dp], ctypes.c_int),
    "lr_cur_id": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, ctypes.c_double,
                   ctypes.c_int, c_ip, c_ip, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_cur_id_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, ctypes.c_double,
                     ctypes.c_int, c_ip, c_ip, c_dp, c_dp, c_dp, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_cur_error_fro": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp],
                         ctypes.c_int),
    "lr_cur_error_fro_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_dp, c_dp, c_dp],
                           ctypes.c_int),
    "lr_read_matrix_binary_d": ([ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_dp,
                                 c_i64], ctypes.c_int),
    "lr_write_matrix_binary_d": ([ctypes.c_void_p, ctypes.c_char_p, c_i64, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_gemm": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_gemm_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_gemm_tn_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64, c_dp, c_i64],
                     ctypes.c_int),
    "lr_randomized_cur_csr_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_ip, c_ip, c_dp, c_i64, lr_sketch_config,
                                 lr_solve_strategy, ctypes.c_double, ctypes.c_int, c_ip, c_ip, c_dp, c_ip, c_ip, c_dp,
                                 c_ip, c_ip, c_dp, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_cur_error_fro_csr_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_ip, c_ip, c_dp, c_i64, c_ip, c_ip, c_dp, c_dp,
                                c_ip, c_ip, c_dp, c_dp], ctypes.c_int),
    "lr_id_from_sample_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, lr_solve_strategy, c_ip, c_dp],
                            ctypes.c_int),
    "lr_tsid_from_skeleton_columns_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, lr_solve_strategy, c_ip, c_dp,
                                         c_dp], ctypes.c_int),
    "lr_gather_columns_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_ip, c_dp, c_i64], ctypes.c_int),
    "lr_gather_rows_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_ip, c_dp, c_i64], ctypes.c_int),
    "lr_transpose_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_cholesky_upper_d": ([ctypes.c_void_p, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_tri_upper_inverse_d": ([ctypes.c_void_p, c_i64, c_dp, c_i64, c_dp, c_i64], ctypes.c_int),
    "lr_cholqr2_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_dp, c_dp, ctypes.POINTER(ctypes.c_int)],
                     ctypes.c_int),
    "lr_residual_norms_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64,
                             ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "lr_error_report_lowrank_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_dp, c_i64, c_dp, c_i64,
                                   ctypes.POINTER(lr_error_report)], ctypes.c_int),
    "lr_verify_lemma1_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, c_dp, c_ip, c_dp, c_dp,
                            ctypes.POINTER(lr_lemma1_report)], ctypes.c_int),
    "lr_verify_lemma2_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, c_dp, c_ip, c_dp,
                            ctypes.POINTER(lr_lemma2_report)], ctypes.c_int),
    "lr_verify_corollary_d": ([ctypes.c_void_p, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, c_dp, c_dp,
                               lr_solve_strategy, ctypes.POINTER(lr_corollary_report)], ctypes.c_int),
    "lr_nccl_get_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "lr_ctx_attach_comm": ([ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "lr_ctx_detach_comm": ([ctypes.c_void_p], ctypes.c_int),
    "lr_ctx_set_shard_emulation": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "lr_ctx_comm_info": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
                         ctypes.c_int),
    "lr_cpqr_sharded_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_i64, c_dp, c_i64, c_i64, c_ip, c_dp],
                          ctypes.c_int),
    "lr_randomized_cur_sharded": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_i64, c_dp, c_i64, c_i64,
                                   lr_sketch_config, lr_solve_strategy, ctypes.c_double, ctypes.c_int, c_ip, c_ip,
                                   c_dp, c_dp, c_dp, c_dp, c_dp, c_dp], ctypes.c_int),
    "lr_randomized_cur_sharded_d": ([ctypes.c_void_p, c_i64, c_i64, c_i64, c_i64, c_dp, c_i64, c_i64,
                                     lr_sketch_config, lr_solve_strategy, ctypes.c_double, ctypes.c_int, c_ip, c_ip,
                                     c_dp, c_dp, c_dp, c_dp, c_dp, c_dp], ctypes.c_int),
}

_lib = None
_lock = threading.Lock()


class LowrankCudaError(RuntimeError):
    """The B200 library or device is unavailable (no CPU fallback exists)."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load liblowrank_b200.so and bind every C-ABI symbol (fails loudly)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise LowrankCudaError(
                f"{path} is missing: build it with __graft_entry__.build() (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib
