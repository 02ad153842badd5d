"""Column-sharded randomized CUR over several GPUs.

Rank g owns a contiguous column block A_g = A(:, off_g : off_g + n_g).  The
pipeline of sketch.hpp:227-234 (+ the lowrank_main.cpp:215 middle factor)
becomes

  stage                        work on rank g                     exchange
  Y_g = Omega A_g              sketch GEMM (Omega from the        -
                               counter stream, identical bits)
  CPQR(Y), l steps             norms, argmax, reflector apply     per step: all-gather of the
                               on the owned columns of Y          N pivot candidates (16 B header
                                                                  + one column each)
  S1 (top k rows of R)         scatter by logical position        all-reduce-sum (exact)
  T = S11^-1 S12               replicated solve                   -
  C = A(:, J)                  masked gather of owned columns     all-reduce-sum (exact)
  CPQR(C^T), k steps           sharded by row blocks of C         as CPQR(Y)
  R_g = A_g(I, :)              local gather                       -
  C = Qc Rc (CholeskyQR2)      replicated                         -
  R^T = Qr Sr                  Gram of R_g^T                      2 x all-reduce (k x k)
  W = Qc^T A Qr                A_g^T Qc, then (.)^T Qr_g           all-reduce (k x k)
  U = Rc^-1 W Sr^-T            replicated                         -

No rank ever holds the whole sample Y: the per-step candidate exchange is
north_star's "NCCL selects the global pivot, the Householder reflector is
broadcast" fused into one all-gather (every rank sends its best column; all
ranks pick the same winner from the same bytes and build the same reflector).

Two implementations of the one protocol:

* the PRODUCT path is native: ``randomized_cur_sharded_device`` is a single
  C-ABI call per rank (``lr_randomized_cur_sharded_d``, csrc/shard.cu +
  csrc/api.cu) over an NCCL communicator the library binds with
  ``attach_nccl`` (unique id shared through torch.distributed);
* ``randomized_cur_sharded`` / ``cpqr_sharded`` below are the same protocol
  step by step on the host over any collective backend -- the executable
  specification the multi-process tests run over gloo on CPU
  (tests/test_distributed.py supplies the shard primitives there; this module
  has no CPU compute of its own).
"""
from __future__ import annotations

import ctypes
from typing import Any, Dict, Optional

import numpy as np


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous column block of rank `rank` (sizes differ by at most one)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi - lo


# ---------------------------------------------------------------- collectives
class TorchComm:
    """Collectives over torch.distributed (gloo on CPU, NCCL for CUDA tensors),
    counting the bytes each rank contributes (tests assert the sample Y is
    never gathered)."""

    def __init__(self, to_tensor, from_tensor):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self._t = to_tensor
        self._f = from_tensor
        self.bytes_sent = 0      # every collective
        self.bytes_gathered = 0  # all-gathers only (the per-step pivot candidates)

    def all_gather_flat(self, x):
        """(L,) on every rank -> (world, L)"""
        import torch
        t = self._t(np.ascontiguousarray(x)).reshape(-1)
        self.bytes_sent += t.numel() * t.element_size()
        self.bytes_gathered += t.numel() * t.element_size()
        if self.world == 1:
            return self._f(t.reshape(1, -1))
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t)
        return self._f(torch.stack(parts))

    def all_reduce_sum(self, x):
        t = self._t(x)
        self.bytes_sent += t.numel() * t.element_size()
        if self.world == 1:
            return x
        tc = t.T.contiguous() if t.dim() == 2 else t.contiguous()
        self.dist.all_reduce(tc)
        return self._f(tc.T if t.dim() == 2 else tc)


# ---------------------------------------------------------------- host protocol
def cpqr_sharded(be, comm, w_local, off: int, n_total: int, steps: int, krows: int):
    """cpqr.hpp:32-114 on the column-sharded short-wide matrix: per step one
    all-gather of the ranks' pivot candidates; the backend applies the
    winner's reflector to the owned columns.  Returns the replicated
    permutation (n_total) and the sign-fixed top `krows` rows of R in logical
    column order (krows x n_total)."""
    st = be.shard_begin(w_local, off)
    for s in range(steps):
        cands = comm.all_gather_flat(be.shard_candidate(st))
        be.shard_step(st, s, cands)
    perm_part, s_part = be.shard_scatter(st, n_total, steps, krows)
    return comm.all_reduce_sum(perm_part), comm.all_reduce_sum(s_part)


def randomized_cur_sharded(be, comm, a_local, col_offset: int, n_total: int, k: int, oversample: int = 10,
                           seed: int = 0, strategy=None) -> Dict[str, Any]:
    """Column-sharded randomized CUR with U = C^+ A R^+ (module docstring), the
    host form of lr_randomized_cur_sharded_d.  Returns the replicated factors
    (C, U, both index sets, both coefficient blocks, skeleton) and this
    rank's block of R."""
    m, n_g = a_local.shape
    ell = k + oversample
    y_local = be.sketch(a_local, ell, seed)
    perm, s1 = cpqr_sharded(be, comm, y_local, col_offset, n_total, min(ell, n_total), k)
    coeff = be.coeff_solve(s1[:, :k], s1[:, k:], strategy)
    own = be.owned_index(perm[:k], col_offset, n_g)
    c = comm.all_reduce_sum(be.gather_columns(a_local, own))
    r0, m_g = shard_bounds(m, comm.world, comm.rank)
    row_perm, s1r = cpqr_sharded(be, comm, be.transpose(c[r0:r0 + m_g, :]), r0, m, k, k)
    row_coeff = be.coeff_solve(s1r[:, :k], s1r[:, k:], strategy)
    skeleton = be.gather_rows(c, row_perm[:k])
    r_local = be.gather_rows(a_local, row_perm[:k])
    # C = Qc Rc (replicated); R^T = Qr Sr by CholeskyQR2 with all-reduced Gram matrices
    rc, rci, ok_c = be.cholqr2(c)
    rt_local = be.transpose(r_local)
    s1g = be.cholesky(comm.all_reduce_sum(be.gemm_tn(rt_local, rt_local)))
    q1_local = be.gemm_tn(r_local, be.tri_inv(s1g))
    s2 = be.cholesky(comm.all_reduce_sum(be.gemm_tn(q1_local, q1_local)))
    sr = be.gemm_tn(be.transpose(s2), s1g)
    sri = be.tri_inv(sr)
    # the same acceptance as the device path: ||Sr||_F ||Sr^-1||_F < min(1e7, 1/threshold)
    ok_r = be.cond_bound(sr, sri) < 1e7
    if not (ok_c and ok_r):
        raise RuntimeError("host protocol: C or R is too ill-conditioned for CholeskyQR2 "
                           "(the device path takes the truncated pseudoinverse route)")
    qr_local = be.gemm_tn(r_local, sri)
    qc = be.gemm_tn(be.transpose(c), rci)
    xt_local = be.gemm_tn(a_local, qc)
    w = comm.all_reduce_sum(be.gemm_tn(xt_local, qr_local))
    t1 = be.gemm_tn(be.transpose(rci), w)
    u = be.gemm_tn(be.transpose(t1), be.transpose(sri))
    return dict(col_pivots=perm, row_pivots=row_perm, c=c, u=u, r_local=r_local, col_coeff=coeff,
                row_coeff=row_coeff, skeleton=skeleton)


# ---------------------------------------------------------------- device (product) path
def attach_nccl(ctx, world: Optional[int] = None, rank: Optional[int] = None) -> None:
    """Bind an NCCL communicator to the library context: rank 0 makes the
    unique id (lr_nccl_get_unique_id), torch.distributed carries it to the
    other ranks, every rank calls lr_ctx_attach_comm.  Without an initialised
    process group (one process) a 1-rank communicator is made."""
    from .lowrank import _raise
    lib = ctx.lib
    if world is None or rank is None:
        try:
            import torch.distributed as dist
            inited = dist.is_initialized()
        except Exception:
            inited = False
        world = dist.get_world_size() if inited else 1
        rank = dist.get_rank() if inited else 0
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        _raise(lib.lr_nccl_get_unique_id(uid))
    if world > 1:
        import torch.distributed as dist
        obj = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = ctypes.create_string_buffer(obj[0], 128)
    _raise(lib.lr_ctx_attach_comm(ctx.h, uid, int(world), int(rank)))


def detach_nccl(ctx) -> None:
    from .lowrank import _raise
    _raise(ctx.lib.lr_ctx_detach_comm(ctx.h))


def randomized_cur_sharded_device(ctx, a_local, col_offset: int, n_total: int, k: int, cfg=None, strategy=None,
                                  pinv_threshold: float = 1e-12, u_mode: Optional[int] = None,
                                  out: Optional[dict] = None) -> dict:
    """lr_randomized_cur_sharded_d: this rank's column block a_local (m x n_g,
    column-major CUDA tensor) of the m x n_total matrix.  Replicated outputs
    (col_pivots, row_pivots, c, u, col_coeff, row_coeff, skeleton) plus r_local
    (k x n_g).  Needs attach_nccl(ctx) on every rank when n_g < n_total."""
    import torch

    from .lowrank import (U_CPINV_A_RPINV, SketchConfig, SolveStrategy, _colmajor_ld, _dptr, _raise,
                          empty_colmajor, on_torch_stream)
    m, n_g = a_local.shape
    dev = a_local.device
    if out is None:
        out = {
            "col_pivots": torch.empty(n_total, dtype=torch.int64, device=dev),
            "row_pivots": torch.empty(m, dtype=torch.int64, device=dev),
            "c": empty_colmajor(m, k, dev), "u": empty_colmajor(k, k, dev),
            "r_local": empty_colmajor(k, max(n_g, 1), dev),
            "col_coeff": empty_colmajor(k, max(n_total - k, 1), dev),
            "row_coeff": empty_colmajor(k, max(m - k, 1), dev), "skeleton": empty_colmajor(k, k, dev),
        }
    with on_torch_stream(ctx):
        _raise(ctx.lib.lr_randomized_cur_sharded_d(
            ctx.h, m, n_g, int(col_offset), int(n_total), _dptr(a_local), _colmajor_ld(a_local), k,
            (cfg or SketchConfig())._c(), (strategy or SolveStrategy.automatic())._c(), float(pinv_threshold),
            int(U_CPINV_A_RPINV if u_mode is None else u_mode), _dptr(out["col_pivots"]), _dptr(out["row_pivots"]),
            _dptr(out["c"]), _dptr(out["u"]), _dptr(out["r_local"]), _dptr(out["col_coeff"]),
            _dptr(out["row_coeff"]), _dptr(out["skeleton"])))
    return out


def randomized_cur_sharded_host(ctx, a_local, col_offset: int, n_total: int, k: int, cfg=None, strategy=None,
                                pinv_threshold: float = 1e-12, u_mode: Optional[int] = None,
                                out: Optional[dict] = None) -> dict:
    """lr_randomized_cur_sharded: this rank's column block in HOST memory (a
    column-major float64 array, ideally page-locked); the upload runs in column
    chunks with each chunk's sketch issued as it lands.  Outputs in host arrays
    (reused from `out`)."""
    from .lowrank import (U_CPINV_A_RPINV, SketchConfig, SolveStrategy, _f64, _ld, _ptr, _raise)
    a_local = _f64(a_local)
    m, n_g = a_local.shape
    if out is None:
        out = {"col_pivots": np.empty(n_total, dtype=np.int64), "row_pivots": np.empty(m, dtype=np.int64),
               "c": np.empty((m, k), order="F"), "u": np.empty((k, k), order="F"),
               "r_local": np.empty((k, n_g), order="F"), "col_coeff": np.empty((k, max(n_total - k, 1)), order="F"),
               "row_coeff": np.empty((k, max(m - k, 1)), order="F"), "skeleton": np.empty((k, k), order="F")}
    _raise(ctx.lib.lr_randomized_cur_sharded(
        ctx.h, m, n_g, int(col_offset), int(n_total), _ptr(a_local), _ld(a_local), k, (cfg or SketchConfig())._c(),
        (strategy or SolveStrategy.automatic())._c(), float(pinv_threshold),
        int(U_CPINV_A_RPINV if u_mode is None else u_mode), _ptr(out["col_pivots"]), _ptr(out["row_pivots"]),
        _ptr(out["c"]), _ptr(out["u"]), _ptr(out["r_local"]), _ptr(out["col_coeff"]), _ptr(out["row_coeff"]),
        _ptr(out["skeleton"])))
    return out


def cpqr_sharded_device(ctx, w_local, col_offset: int, n_total: int, k: int):
    """lr_cpqr_sharded_d: pivots (n_total) and the sign-fixed top k rows of R in
    logical order (k x n_total), replicated."""
    import torch

    from .lowrank import _colmajor_ld, _dptr, _raise, empty_colmajor, on_torch_stream
    m, n_g = w_local.shape
    piv = torch.empty(n_total, dtype=torch.int64, device=w_local.device)
    s = empty_colmajor(k, n_total, w_local.device)
    with on_torch_stream(ctx):
        _raise(ctx.lib.lr_cpqr_sharded_d(ctx.h, m, n_g, int(col_offset), int(n_total), _dptr(w_local),
                                         _colmajor_ld(w_local), k, _dptr(piv), _dptr(s)))
    return piv, s


def set_shard_emulation(ctx, nshards: int) -> None:
    """Single-GPU test vehicle: without a communicator, run the sharded CPQRs as
    `nshards` column blocks in this process (lr_ctx_set_shard_emulation)."""
    from .lowrank import _raise
    _raise(ctx.lib.lr_ctx_set_shard_emulation(ctx.h, int(nshards)))
