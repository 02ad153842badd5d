"""Python mirror of the reference ``lowrank`` API, running on the B200 C ABI.

Names, argument meaning, defaults and error classes follow
/root/reference/proj/include/lowrank (cited per function); matrices are
numpy float64 arrays (any layout; copied to column-major) and index vectors
are int64.  Every compute call goes through ``liblowrank_b200.so`` -- there
is no CPU path.  ``*_device`` variants take torch CUDA tensors (column-major,
i.e. ``t.T.contiguous().T`` / ``torch.empty((n, m)).T``) and return device
tensors; they are what bench.py times.
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

__all__ = [
    "SingularityError", "ConvergenceError", "LowrankCudaError", "SolveKind", "SolveStrategy", "SketchKind",
    "SketchConfig", "PivotedQr", "ColumnId", "RowId", "TwoSidedId", "CurDecomposition", "SampleMatrix",
    "Context", "default_context", "gaussian_matrix", "sketch_gaussian", "sketch_srft", "srft_operator", "sketch_power", "cpqr_partial", "cpqr_full",
    "stabilized_coeff_solve", "svd", "pinv", "id_column", "id_row", "tsid_from_column_id", "id_two_sided",
    "cur_from_two_sided", "cur_id", "randomized_id", "randomized_cur", "randomized_svd", "select_columns", "select_rows",
    "skeleton_columns", "skeleton_rows", "reconstruct", "frobenius_norm", "cur_error_fro",
    "randomized_cur_device", "cur_error_fro_device", "empty_colmajor", "U_VT_RPINV", "U_CPINV_A_RPINV",
    "randomized_cur_csr_device", "cur_error_fro_csr_device", "pinned_cur_outputs", "CUR_OUTPUT_KEYS",
    "id_column_device", "randomized_id_device", "cur_id_device", "residual_norms_device", "matmul", "error_report_device",
    "verify_lemma1_device", "verify_lemma2_device", "verify_corollary_device", "ParseError",
    "read_matrix_binary_device", "write_matrix_binary_device",
]

LowrankCudaError = L.LowrankCudaError
U_VT_RPINV = L.LR_U_VT_RPINV          # cur.hpp:30
U_CPINV_A_RPINV = L.LR_U_CPINV_A_RPINV  # lowrank_main.cpp:215


class ParseError(RuntimeError):
    """core.hpp:40-42: malformed input file (io.hpp readers)."""


class SingularityError(RuntimeError):
    """core.hpp:24-32: zero diagonal with an inconsistent right-hand side."""

    def __init__(self, what: str, index: int):
        super().__init__(what)
        self._index = index

    def index(self) -> int:
        return self._index


class ConvergenceError(RuntimeError):
    """core.hpp:35-37: Jacobi sweep cap exhausted."""


def _raise(rc: int) -> None:
    if rc == L.LR_OK:
        return
    lib = L.load()
    msg = (lib.lr_last_error() or b"").decode()
    if rc == L.LR_EINVAL:
        raise ValueError(msg)
    if rc == L.LR_ESINGULAR:
        raise SingularityError(msg, int(lib.lr_last_singular_index()))
    if rc == L.LR_ECONVERGE:
        raise ConvergenceError(msg)
    if rc == L.LR_ECUDA:
        raise LowrankCudaError(msg)
    if rc == L.LR_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == L.LR_EPARSE:
        raise ParseError(msg)
    raise RuntimeError(msg)


# ------------------------------------------------------------------ configs
class SolveKind:
    BackSubstitution = L.LR_SOLVE_BACKSUB
    TruncatedPinv = L.LR_SOLVE_PINV
    Tikhonov = L.LR_SOLVE_TIKHONOV


@dataclass
class SolveStrategy:
    """solve.hpp:16-32 (defaults: back-substitution, 1e-12, escalate)."""
    kind: int = SolveKind.BackSubstitution
    threshold: float = 1e-12
    ridge: float = 0.0
    escalate: bool = True

    @staticmethod
    def automatic() -> "SolveStrategy":
        return SolveStrategy()

    @staticmethod
    def back_substitution(threshold: float = 1e-12) -> "SolveStrategy":
        return SolveStrategy(SolveKind.BackSubstitution, threshold, 0.0, False)

    @staticmethod
    def truncated_pinv(threshold: float = 1e-12) -> "SolveStrategy":
        return SolveStrategy(SolveKind.TruncatedPinv, threshold, 0.0, False)

    @staticmethod
    def tikhonov(ridge: float, threshold: float = 1e-12) -> "SolveStrategy":
        return SolveStrategy(SolveKind.Tikhonov, threshold, ridge, False)

    def _c(self) -> L.lr_solve_strategy:
        return L.lr_solve_strategy(int(self.kind), float(self.threshold), float(self.ridge), int(bool(self.escalate)))


class SketchKind:
    Gaussian = L.LR_SKETCH_GAUSSIAN
    Srft = L.LR_SKETCH_SRFT


@dataclass
class SketchConfig:
    """sketch.hpp:21-33 (defaults: Gaussian, p = 10, q = 0, seed 0)."""
    kind: int = SketchKind.Gaussian
    oversample: int = 10
    srft_samples: int = 0
    power: int = 0
    reorthonormalize: bool = True
    seed: int = 0

    def sample_count(self, k: int) -> int:
        if self.kind == SketchKind.Gaussian:
            return k + int(self.oversample)
        return self.srft_samples if self.srft_samples > 0 else 2 * k

    def _c(self) -> L.lr_sketch_config:
        return L.lr_sketch_config(int(self.kind), int(self.oversample), int(self.srft_samples), int(self.power),
                                  int(bool(self.reorthonormalize)), int(self.seed) & 0xFFFFFFFFFFFFFFFF)


# ------------------------------------------------------------------ results
@dataclass
class PivotedQr:
    """cpqr.hpp:15-21."""
    q: Optional[np.ndarray]
    s: np.ndarray
    pivots: np.ndarray
    rank_achieved: int = 0


@dataclass
class ColumnId:
    """id.hpp:12-31."""
    cols: int
    rank: int
    pivots: np.ndarray
    coeff: np.ndarray

    def basis(self) -> np.ndarray:
        v = np.zeros((self.cols, self.rank), order="F")
        v[self.pivots[: self.rank], np.arange(self.rank)] = 1.0
        v[self.pivots[self.rank:], :] = self.coeff.T
        return v


@dataclass
class RowId:
    """id.hpp:34-53."""
    rows: int
    rank: int
    pivots: np.ndarray
    coeff: np.ndarray

    def basis(self) -> np.ndarray:
        w = np.zeros((self.rows, self.rank), order="F")
        w[self.pivots[: self.rank], np.arange(self.rank)] = 1.0
        w[self.pivots[self.rank:], :] = self.coeff.T
        return w


@dataclass
class TwoSidedId:
    """id.hpp:59-70."""
    col_id: ColumnId
    row_id: RowId
    skeleton: np.ndarray

    def col_pivots(self) -> np.ndarray:
        return self.col_id.pivots

    def row_pivots(self) -> np.ndarray:
        return self.row_id.pivots

    def col_basis(self) -> np.ndarray:
        return self.col_id.basis()

    def row_basis(self) -> np.ndarray:
        return self.row_id.basis()

    def rank(self) -> int:
        return self.col_id.rank


@dataclass
class CurDecomposition:
    """cur.hpp:9-18."""
    c: np.ndarray
    u: np.ndarray
    r: np.ndarray
    col_pivots: np.ndarray
    row_pivots: np.ndarray

    def rank(self) -> int:
        return self.u.shape[0]


@dataclass
class SampleProvenance:
    kind: int = SketchKind.Gaussian
    samples: int = 0
    power: int = 0
    reorthonormalized: bool = False
    seed: int = 0


@dataclass
class SampleMatrix:
    """sketch.hpp:36-50."""
    y: np.ndarray
    provenance: SampleProvenance = field(default_factory=SampleProvenance)


# ------------------------------------------------------------------ context
class Context:
    """An lr_ctx: one device, one stream, cached workspaces."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = ctypes.c_void_p()
        _raise(self.lib.lr_ctx_create(ctypes.byref(h), int(device)))
        self.h = h
        self.device = device
        self._stream = None  # None: the context's own stream

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.lr_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int) -> None:
        """Run subsequent device calls on this cudaStream_t (0 = the legacy default stream)."""
        _raise(self.lib.lr_ctx_set_stream(self.h, ctypes.c_void_p(stream_handle)))
        self._stream = stream_handle

    def use_own_stream(self) -> None:
        _raise(self.lib.lr_ctx_use_own_stream(self.h))
        self._stream = None

    GEMM_DMMA = 0
    GEMM_OZAKI_INT8 = 1

    def set_gemm_mode(self, mode: int) -> None:
        """Engine of the A-sized contractions: GEMM_DMMA (FP64 tensor cores,
        default) or GEMM_OZAKI_INT8 (FP64 emulated on the INT8 tensor cores)."""
        _raise(self.lib.lr_ctx_set_gemm_mode(self.h, int(mode)))

    def set_concurrent_tail(self, sms: int = -1) -> None:
        """Schedule of the randomized CUR's tail: sms > 0 runs the row ID of C
        on an SM partition of that size next to A^T Q_c, 0 runs them one after
        the other, -1 (default) lets the library choose."""
        _raise(self.lib.lr_ctx_set_concurrent_tail(self.h, int(sms)))

    def gemm_mode(self) -> int:
        return int(self.lib.lr_ctx_get_gemm_mode(self.h))

    def stats(self) -> dict:
        st = L.lr_stats()
        _raise(self.lib.lr_ctx_get_stats(self.h, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in L.lr_stats._fields_}

    def synchronize(self) -> None:
        _raise(self.lib.lr_ctx_synchronize(self.h))

    def enable_timing(self, on: bool = True) -> None:
        _raise(self.lib.lr_ctx_enable_timing(self.h, int(on)))

    def stage_report(self) -> dict:
        import json
        buf = ctypes.create_string_buffer(1 << 16)
        _raise(self.lib.lr_ctx_stage_report(self.h, buf, len(buf)))
        return json.loads(buf.value.decode())

    def release_workspace(self) -> None:
        """Free the grow-only device workspace (Ozaki residue planes, CPQR state, call arena)."""
        _raise(self.lib.lr_ctx_release_workspace(self.h))

    def reset_stats(self) -> None:
        _raise(self.lib.lr_ctx_reset_stats(self.h))

    def kernel_launches(self) -> int:
        return int(self.lib.lr_kernel_launches())


_default: Optional[Context] = None


@contextlib.contextmanager
def on_torch_stream(c: "Context"):
    """Device entry points called on torch tensors run in torch's current
    stream order (inputs written and outputs allocated by torch are then
    ordered with the library's kernels), unless the context was bound to a
    stream explicitly with set_stream."""
    if c._stream is not None:
        yield
        return
    import torch
    c.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        yield
    finally:
        c.use_own_stream()


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _f64(a) -> np.ndarray:
    """float64 column-major input; a column-major view with a padded leading
    dimension (e.g. big[:m] of a Fortran array) is passed through uncopied."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2 and a.strides[0] == 8 and a.strides[1] % 8 == 0 and a.strides[1] >= 8 * max(1, a.shape[0]):
        return a
    return np.asfortranarray(a)


def _fc(a) -> np.ndarray:
    """compact column-major float64 (arrays the ABI takes without a leading dimension)"""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _ptr(x: np.ndarray) -> int:
    return x.ctypes.data


def _ld(a: np.ndarray) -> int:
    """leading dimension (elements between columns) of a column-major array"""
    if a.ndim == 2 and a.shape[1] > 1 and a.strides[0] == 8:
        return max(1, a.strides[1] // 8, a.shape[0])
    return max(1, a.shape[0])


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else default_context()


# ------------------------------------------------------------------ rng / sketch
def gaussian_matrix(rows: int, cols: int, seed: int, ctx: Optional[Context] = None) -> np.ndarray:
    """rng.hpp:74-94 (generated on the GPU)."""
    c = _ctx(ctx)
    out = np.empty((max(rows, 0), max(cols, 0)), order="F")
    _raise(c.lib.lr_gaussian_matrix(c.h, rows, cols, int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(out)))
    return out


def sketch_gaussian(a, ell: int, seed: int, ctx: Optional[Context] = None) -> SampleMatrix:
    """sketch.hpp:67-78: Y = Omega A."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    y = np.empty((max(ell, 0), n), order="F")
    _raise(c.lib.lr_sketch_gaussian(c.h, m, n, _ptr(a), _ld(a), ell, int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(y)))
    return SampleMatrix(y, SampleProvenance(SketchKind.Gaussian, ell, 0, False, seed))


# ------------------------------------------------------------------ CPQR / solve / SVD
def randomized_svd(a, k: int, cfg: Optional[SketchConfig] = None, ctx: Optional[Context] = None) -> Svd:
    """sketch.hpp:238-254: orth_rows of the sample, SVD of A Q^T, truncated to rank k."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 1)
    u = np.empty((m, kk), order="F")
    s = np.empty(kk)
    v = np.empty((n, kk), order="F")
    _raise(c.lib.lr_randomized_svd(c.h, m, n, _ptr(a), _ld(a), int(k), (cfg or SketchConfig())._c(), _ptr(u), _ptr(s),
                                   _ptr(v)))
    return Svd(u, s, v)


def sketch_srft(a, ell: int, seed: int, ctx: Optional[Context] = None) -> SampleMatrix:
    """sketch.hpp:110-143: sqrt(m/ell) R H D A (subsampled randomized Hartley transform)."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    y = np.empty((int(ell), n), order="F")
    _raise(c.lib.lr_sketch_srft(c.h, m, n, _ptr(a), _ld(a), int(ell), int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(y)))
    return SampleMatrix(y, SampleProvenance(SketchKind.Srft, int(ell), 0, False, int(seed)))


def srft_operator(m: int, ell: int, seed: int, ctx: Optional[Context] = None) -> np.ndarray:
    """sketch.hpp:84-100: the dense SRFT operator sqrt(m/ell) R H D (ell x m)."""
    c = _ctx(ctx)
    out = np.empty((int(ell), int(m)), order="F")
    _raise(c.lib.lr_srft_operator(c.h, int(m), int(ell), int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(out)))
    return out


def sketch_power(a, ell: int, q: int, reorthonormalize: bool = True, seed: int = 0,
                 ctx: Optional[Context] = None) -> SampleMatrix:
    """sketch.hpp:148-164: Omega A (A^T A)^q (rows re-orthonormalised before each product)."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    y = np.zeros((int(ell), n), order="F")
    rows = ctypes.c_int64(0)
    _raise(c.lib.lr_sketch_power(c.h, m, n, _ptr(a), _ld(a), int(ell), int(q), int(bool(reorthonormalize)),
                                 int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(y), ctypes.byref(rows)))
    prov = SampleProvenance(SketchKind.Gaussian, int(ell), int(q), bool(reorthonormalize) and q > 0, int(seed))
    return SampleMatrix(np.asfortranarray(y[: rows.value]), prov)


def cpqr_partial(a, k: int, want_q: bool = True, ctx: Optional[Context] = None) -> PivotedQr:
    """cpqr.hpp:32-114."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 0)
    s = np.empty((kk, n), order="F")
    q = np.empty((m, kk), order="F") if want_q else None
    piv = np.empty(n, dtype=np.int64)
    _raise(c.lib.lr_cpqr_partial(c.h, m, n, _ptr(a), _ld(a), k, _ptr(q) if q is not None else None, _ptr(s),
                                 _ptr(piv)))
    return PivotedQr(q, s, piv, int(k))


def cpqr_full(a, want_q: bool = True, ctx: Optional[Context] = None) -> PivotedQr:
    """cpqr.hpp:118-122."""
    a = _f64(a)
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("cpqr_full: matrix must be nonempty")
    return cpqr_partial(a, min(a.shape), want_q, ctx)


def stabilized_coeff_solve(s11, s12, strategy: Optional[SolveStrategy] = None,
                           ctx: Optional[Context] = None) -> np.ndarray:
    """solve.hpp:104-145."""
    c = _ctx(ctx)
    s11 = _f64(s11)
    s12 = _f64(s12)
    if s11.ndim != 2 or s11.shape[0] != s11.shape[1]:
        raise ValueError("stabilized_coeff_solve: triangular block must be square")
    if s12.shape[0] != s11.shape[0]:
        raise ValueError("stabilized_coeff_solve: row count mismatch")
    k, nc = s12.shape
    t = np.empty((k, nc), order="F")
    st = (strategy or SolveStrategy.automatic())._c()
    _raise(c.lib.lr_stabilized_coeff_solve(c.h, k, nc, _ptr(s11), _ld(s11), _ptr(s12), _ld(s12), st, _ptr(t)))
    return t


@dataclass
class Svd:
    """svd.hpp:16-28."""
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray

    def rank(self, rel_threshold: float) -> int:
        if self.sigma.size == 0 or self.sigma[0] == 0.0:
            return 0
        return int(np.count_nonzero(self.sigma >= rel_threshold * self.sigma[0]))


def svd(a, ctx: Optional[Context] = None) -> Svd:
    """svd.hpp:132-183 (one-sided Jacobi on the GPU)."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    r = min(m, n)
    u = np.empty((m, r), order="F")
    s = np.empty(r)
    v = np.empty((n, r), order="F")
    _raise(c.lib.lr_svd(c.h, m, n, _ptr(a), _ld(a), _ptr(u), _ptr(s), _ptr(v)))
    return Svd(u, s, v)


def pinv(a, threshold: float = 1e-12, ctx: Optional[Context] = None) -> np.ndarray:
    """svd.hpp:193-207."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    out = np.empty((n, m), order="F")
    _raise(c.lib.lr_pinv(c.h, m, n, _ptr(a), _ld(a), float(threshold), _ptr(out)))
    return out


# ------------------------------------------------------------------ ID / CUR
def id_column(a, k: int, strategy: Optional[SolveStrategy] = None, ctx: Optional[Context] = None) -> ColumnId:
    """id.hpp:91-105."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 0)
    piv = np.empty(n, dtype=np.int64)
    coeff = np.empty((kk, max(n - kk, 0)), order="F")
    st = (strategy or SolveStrategy.automatic())._c()
    _raise(c.lib.lr_id_column(c.h, m, n, _ptr(a), _ld(a), k, st, _ptr(piv), _ptr(coeff)))
    return ColumnId(n, int(k), piv, coeff)


def id_row(a, k: int, strategy: Optional[SolveStrategy] = None, ctx: Optional[Context] = None) -> RowId:
    """id.hpp:108-119."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 0)
    piv = np.empty(m, dtype=np.int64)
    coeff = np.empty((kk, max(m - kk, 0)), order="F")
    st = (strategy or SolveStrategy.automatic())._c()
    _raise(c.lib.lr_id_row(c.h, m, n, _ptr(a), _ld(a), k, st, _ptr(piv), _ptr(coeff)))
    return RowId(m, int(k), piv, coeff)


def tsid_from_column_id(a, col_id: ColumnId, strategy: Optional[SolveStrategy] = None,
                        ctx: Optional[Context] = None) -> TwoSidedId:
    """id.hpp:124-134."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    k = col_id.rank
    cp = np.ascontiguousarray(col_id.pivots, dtype=np.int64)
    rp = np.empty(m, dtype=np.int64)
    rc = np.empty((k, max(m - k, 0)), order="F")
    sk = np.empty((k, k), order="F")
    st = (strategy or SolveStrategy.automatic())._c()
    _raise(c.lib.lr_tsid_from_column_id(c.h, m, n, _ptr(a), _ld(a), k, _ptr(cp), st, _ptr(rp), _ptr(rc),
                                        _ptr(sk)))
    return TwoSidedId(col_id, RowId(m, k, rp, rc), sk)


def id_two_sided(a, k: int, strategy: Optional[SolveStrategy] = None, ctx: Optional[Context] = None) -> TwoSidedId:
    """id.hpp:137-141."""
    return tsid_from_column_id(a, id_column(a, k, strategy, ctx), strategy, ctx)


def cur_from_two_sided(a, tsid: TwoSidedId, pinv_threshold: float = 1e-12, u_mode: int = U_VT_RPINV,
                       ctx: Optional[Context] = None) -> CurDecomposition:
    """cur.hpp:23-34 (u_mode U_VT_RPINV) / lowrank_main.cpp:210-215 (U_CPINV_A_RPINV)."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    k = tsid.rank()
    cp = np.ascontiguousarray(tsid.col_pivots(), dtype=np.int64)
    rp = np.ascontiguousarray(tsid.row_pivots(), dtype=np.int64)
    cc = _fc(tsid.col_id.coeff)
    C = np.empty((m, k), order="F")
    U = np.empty((k, k), order="F")
    R = np.empty((k, n), order="F")
    _raise(c.lib.lr_cur_from_two_sided(c.h, m, n, _ptr(a), _ld(a), k, _ptr(cp), _ptr(cc), _ptr(rp),
                                       float(pinv_threshold), int(u_mode), _ptr(C), _ptr(U), _ptr(R)))
    return CurDecomposition(C, U, R, cp.copy(), rp.copy())


CUR_OUTPUT_KEYS = ("col_pivots", "row_pivots", "c", "u", "r", "col_coeff", "row_coeff", "skeleton")


def _cur_shapes(m, n, k):
    return ((n,), (m,), (m, k), (k, k), (k, n), (k, max(n - k, 0)), (k, max(m - k, 0)), (k, k))


def _cur_outputs(m, n, k, out=None):
    if out is not None:
        arrs = tuple(out[key] for key in CUR_OUTPUT_KEYS)
        for key, arr, shp in zip(CUR_OUTPUT_KEYS, arrs, _cur_shapes(m, n, k)):
            want = np.int64 if key.endswith("pivots") else np.float64
            if arr.shape != shp or arr.dtype != want or not (arr.ndim == 1 or arr.flags.f_contiguous):
                raise ValueError(f"out['{key}']: expected a {shp} column-major {np.dtype(want).name} array")
        return arrs
    return (np.empty(n, dtype=np.int64), np.empty(m, dtype=np.int64), np.empty((m, k), order="F"),
            np.empty((k, k), order="F"), np.empty((k, n), order="F"), np.empty((k, max(n - k, 0)), order="F"),
            np.empty((k, max(m - k, 0)), order="F"), np.empty((k, k), order="F"))


def pinned_cur_outputs(m: int, n: int, k: int) -> dict:
    """Page-locked host buffers for randomized_cur(..., out=): the factors are
    then copied back on a separate stream while the rest of the CUR runs."""
    import torch
    out = {}
    for key, shp in zip(CUR_OUTPUT_KEYS, _cur_shapes(m, n, k)):
        if key.endswith("pivots"):
            out[key] = torch.empty(shp, dtype=torch.int64, pin_memory=True).numpy()
        else:
            out[key] = torch.empty(shp[::-1], dtype=torch.float64, pin_memory=True).numpy().T
    return out


def cur_id(a, k: int, strategy: Optional[SolveStrategy] = None, pinv_threshold: float = 1e-12,
           u_mode: int = U_VT_RPINV, ctx: Optional[Context] = None, return_tsid: bool = False):
    """cur.hpp:37-42 (deterministic CUR via the two-sided ID)."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 1)
    cp, rp, C, U, R, cc, rc, sk = _cur_outputs(m, n, kk)
    st = (strategy or SolveStrategy.automatic())._c()
    _raise(c.lib.lr_cur_id(c.h, m, n, _ptr(a), _ld(a), k, st, float(pinv_threshold), int(u_mode), _ptr(cp),
                           _ptr(rp), _ptr(C), _ptr(U), _ptr(R), _ptr(cc), _ptr(rc), _ptr(sk)))
    cur = CurDecomposition(C, U, R, cp, rp)
    if return_tsid:
        return cur, TwoSidedId(ColumnId(n, k, cp, cc), RowId(m, k, rp, rc), sk)
    return cur


def randomized_id(a, k: int, cfg: Optional[SketchConfig] = None, strategy: Optional[SolveStrategy] = None,
                  ctx: Optional[Context] = None) -> ColumnId:
    """sketch.hpp:200-223."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 0)
    piv = np.empty(n, dtype=np.int64)
    coeff = np.empty((kk, max(n - kk, 0)), order="F")
    _raise(c.lib.lr_randomized_id(c.h, m, n, _ptr(a), _ld(a), k, (cfg or SketchConfig())._c(),
                                  (strategy or SolveStrategy.automatic())._c(), _ptr(piv), _ptr(coeff)))
    return ColumnId(n, int(k), piv, coeff)


def randomized_cur(a, k: int, cfg: Optional[SketchConfig] = None, strategy: Optional[SolveStrategy] = None,
                   pinv_threshold: float = 1e-12, u_mode: int = U_VT_RPINV, ctx: Optional[Context] = None,
                   return_tsid: bool = False, out: Optional[dict] = None):
    """sketch.hpp:227-234 (+ the lowrank_main.cpp:215 middle factor with U_CPINV_A_RPINV).
    `out`: preallocated outputs (e.g. pinned_cur_outputs) reused across calls."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    kk = max(int(k), 1)
    cp, rp, C, U, R, cc, rc, sk = _cur_outputs(m, n, kk, out if int(k) >= 1 else None)
    _raise(c.lib.lr_randomized_cur(c.h, m, n, _ptr(a), _ld(a), k, (cfg or SketchConfig())._c(),
                                   (strategy or SolveStrategy.automatic())._c(), float(pinv_threshold), int(u_mode),
                                   _ptr(cp), _ptr(rp), _ptr(C), _ptr(U), _ptr(R), _ptr(cc), _ptr(rc), _ptr(sk)))
    cur = CurDecomposition(C, U, R, cp, rp)
    if return_tsid:
        return cur, TwoSidedId(ColumnId(n, k, cp, cc), RowId(m, k, rp, rc), sk)
    return cur


def cur_error_fro(a, cur: CurDecomposition, ctx: Optional[Context] = None):
    """(||A - C U R||_F, ||A||_F) computed by the fused DMMA residual kernel."""
    c = _ctx(ctx)
    a = _f64(a)
    m, n = a.shape
    k = cur.rank()
    out = np.empty(2)
    C, U, R = _fc(cur.c), _fc(cur.u), _fc(cur.r)
    _raise(c.lib.lr_cur_error_fro(c.h, m, n, _ptr(a), _ld(a), k, _ptr(C), _ptr(U), _ptr(R), _ptr(out)))
    return float(out[0]), float(out[1])


# ------------------------------------------------------------------ small host helpers (core.hpp / id.hpp)
def select_columns(a, pivots, count: int) -> np.ndarray:
    """core.hpp:70-76 (a gather; the device path gathers on the GPU)."""
    return np.asfortranarray(np.asarray(a)[:, np.asarray(pivots)[:count]])


def select_rows(a, pivots, count: int) -> np.ndarray:
    """core.hpp:79-85."""
    return np.asfortranarray(np.asarray(a)[np.asarray(pivots)[:count], :])


def skeleton_columns(a, cid: ColumnId) -> np.ndarray:
    return select_columns(a, cid.pivots, cid.rank)


def skeleton_rows(a, rid: RowId) -> np.ndarray:
    return select_rows(a, rid.pivots, rid.rank)


def matmul(a, b, ctx: Optional[Context] = None) -> np.ndarray:
    """C = A B on the GPU (lr_gemm, FP64 DMMA): the products of the reconstructions."""
    c = _ctx(ctx)
    a, b = _f64(a), _f64(b)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("matmul: inner dimensions differ")
    out = np.empty((m, n), order="F")
    if m == 0 or n == 0:
        return out
    if k == 0:
        out[:] = 0.0
        return out
    _raise(c.lib.lr_gemm(c.h, m, n, k, _ptr(a), _ld(a), _ptr(b), _ld(b), _ptr(out), max(1, m)))
    return out


def reconstruct(*args):
    """id.hpp:144-159 / cur.hpp:77-80, the products on the GPU (lr_gemm)."""
    if len(args) == 1 and isinstance(args[0], CurDecomposition):
        cur = args[0]
        return matmul(matmul(cur.c, cur.u), cur.r)
    if len(args) == 1 and isinstance(args[0], TwoSidedId):
        t = args[0]
        return matmul(matmul(t.row_basis(), t.skeleton), np.asfortranarray(t.col_basis().T))
    a, idobj = args
    if isinstance(idobj, ColumnId):
        return matmul(skeleton_columns(a, idobj), np.asfortranarray(idobj.basis().T))
    return matmul(idobj.basis(), skeleton_rows(a, idobj))


def frobenius_norm(a) -> float:
    """core.hpp:64-67."""
    return float(np.linalg.norm(np.asarray(a)))


# ------------------------------------------------------------------ device (torch) entry points
def _dptr(t) -> int:
    return int(t.data_ptr())


def _colmajor_ld(t) -> int:
    # a column-major (m x n) torch tensor has stride (1, ld)
    if t.dim() != 2 or t.stride(0) != 1:
        raise ValueError("expected a column-major 2-D tensor (stride(0) == 1)")
    return int(t.stride(1)) if t.shape[1] > 1 else max(1, int(t.shape[0]))


def empty_colmajor(m: int, n: int, device, dtype=None):
    import torch
    return torch.empty((n, m), device=device, dtype=dtype or torch.float64).T


def randomized_cur_device(a, k: int, cfg: Optional[SketchConfig] = None, strategy: Optional[SolveStrategy] = None,
                          pinv_threshold: float = 1e-12, u_mode: int = U_CPINV_A_RPINV,
                          ctx: Optional[Context] = None, out: Optional[dict] = None) -> dict:
    """lr_randomized_cur_d on a device-resident column-major tensor."""
    import torch
    c = _ctx(ctx)
    m, n = a.shape
    lda = _colmajor_ld(a)
    dev = a.device
    if out is None:
        out = {
            "col_pivots": torch.empty(n, dtype=torch.int64, device=dev),
            "row_pivots": torch.empty(m, dtype=torch.int64, device=dev),
            "c": empty_colmajor(m, k, dev), "u": empty_colmajor(k, k, dev), "r": empty_colmajor(k, n, dev),
            "col_coeff": empty_colmajor(k, max(n - k, 1), dev), "row_coeff": empty_colmajor(k, max(m - k, 1), dev),
            "skeleton": empty_colmajor(k, k, dev),
        }
    with on_torch_stream(c):
        _raise(c.lib.lr_randomized_cur_d(
            c.h, m, n, _dptr(a), lda, k, (cfg or SketchConfig())._c(), (strategy or SolveStrategy.automatic())._c(),
            float(pinv_threshold), int(u_mode), _dptr(out["col_pivots"]), _dptr(out["row_pivots"]), _dptr(out["c"]),
            _dptr(out["u"]), _dptr(out["r"]), _dptr(out["col_coeff"]), _dptr(out["row_coeff"]),
            _dptr(out["skeleton"])))
    return out


def id_column_device(a, k: int, strategy: Optional[SolveStrategy] = None, ctx: Optional[Context] = None,
                     out: Optional[dict] = None) -> dict:
    """lr_id_column_d (id.hpp:91-105) on a device-resident column-major tensor."""
    import torch
    c = _ctx(ctx)
    m, n = a.shape
    if out is None:
        out = {"pivots": torch.empty(n, dtype=torch.int64, device=a.device),
               "coeff": empty_colmajor(k, max(n - k, 1), a.device)}
    with on_torch_stream(c):
        _raise(c.lib.lr_id_column_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k,
                                    (strategy or SolveStrategy.automatic())._c(), _dptr(out["pivots"]),
                                    _dptr(out["coeff"])))
    return out


def randomized_id_device(a, k: int, cfg: Optional[SketchConfig] = None, strategy: Optional[SolveStrategy] = None,
                         ctx: Optional[Context] = None, out: Optional[dict] = None) -> dict:
    """lr_randomized_id_d (sketch.hpp:200-223) on a device-resident column-major tensor."""
    import torch
    c = _ctx(ctx)
    m, n = a.shape
    if out is None:
        out = {"pivots": torch.empty(n, dtype=torch.int64, device=a.device),
               "coeff": empty_colmajor(k, max(n - k, 1), a.device)}
    with on_torch_stream(c):
        _raise(c.lib.lr_randomized_id_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, (cfg or SketchConfig())._c(),
                                        (strategy or SolveStrategy.automatic())._c(), _dptr(out["pivots"]),
                                        _dptr(out["coeff"])))
    return out


def cur_id_device(a, k: int, strategy: Optional[SolveStrategy] = None, pinv_threshold: float = 1e-12,
                  u_mode: int = U_VT_RPINV, ctx: Optional[Context] = None, out: Optional[dict] = None) -> dict:
    """lr_cur_id_d (cur.hpp:36-42; U = C^+ A R^+ with U_CPINV_A_RPINV) on a
    device-resident column-major tensor."""
    import torch
    c = _ctx(ctx)
    m, n = a.shape
    dev = a.device
    if out is None:
        out = {
            "col_pivots": torch.empty(n, dtype=torch.int64, device=dev),
            "row_pivots": torch.empty(m, dtype=torch.int64, device=dev),
            "c": empty_colmajor(m, k, dev), "u": empty_colmajor(k, k, dev), "r": empty_colmajor(k, n, dev),
            "col_coeff": empty_colmajor(k, max(n - k, 1), dev), "row_coeff": empty_colmajor(k, max(m - k, 1), dev),
            "skeleton": empty_colmajor(k, k, dev),
        }
    with on_torch_stream(c):
        _raise(c.lib.lr_cur_id_d(
            c.h, m, n, _dptr(a), _colmajor_ld(a), k, (strategy or SolveStrategy.automatic())._c(),
            float(pinv_threshold), int(u_mode), _dptr(out["col_pivots"]), _dptr(out["row_pivots"]), _dptr(out["c"]),
            _dptr(out["u"]), _dptr(out["r"]), _dptr(out["col_coeff"]), _dptr(out["row_coeff"]),
            _dptr(out["skeleton"])))
    return out


def cur_error_fro_device(a, cur: dict, ctx: Optional[Context] = None):
    c = _ctx(ctx)
    m, n = a.shape
    k = cur["u"].shape[0]
    res = np.empty(2)
    with on_torch_stream(c):
        _raise(c.lib.lr_cur_error_fro_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, _dptr(cur["c"]), _dptr(cur["u"]),
                                        _dptr(cur["r"]), _ptr(res)))
    return float(res[0]), float(res[1])


# ------------------------------------------------------------------ io.hpp binary matrices <-> device
def read_matrix_binary_device(path: str, device="cuda", ctx: Optional[Context] = None):
    """io.hpp:215-233 read_matrix_binary straight into a column-major CUDA tensor
    (row blocks streamed through page-locked buffers, transposed on the GPU)."""
    c = _ctx(ctx)
    rows, cols = ctypes.c_int64(0), ctypes.c_int64(0)
    _raise(c.lib.lr_read_matrix_binary_d(c.h, str(path).encode(), ctypes.byref(rows), ctypes.byref(cols), None, 1))
    out = empty_colmajor(rows.value, cols.value, device)
    with on_torch_stream(c):
        _raise(c.lib.lr_read_matrix_binary_d(c.h, str(path).encode(), ctypes.byref(rows), ctypes.byref(cols),
                                             _dptr(out), _colmajor_ld(out)))
    return out


def write_matrix_binary_device(path: str, a, ctx: Optional[Context] = None) -> None:
    """io.hpp:199-213 write_matrix_binary from a column-major CUDA tensor."""
    c = _ctx(ctx)
    m, n = a.shape
    with on_torch_stream(c):
        _raise(c.lib.lr_write_matrix_binary_d(c.h, str(path).encode(), m, n, _dptr(a), _colmajor_ld(a)))


# ------------------------------------------------------------------ verifiers at scale (verify.hpp)
def _rep(st) -> dict:
    return {f: (bool(getattr(st, f)) if t is ctypes.c_int else float(getattr(st, f))) for f, t in st._fields_}


def residual_norms_device(a, x=None, y=None, spectral: bool = True, ctx: Optional[Context] = None):
    """(||A - X Y||_2, ||A - X Y||_F) for device tensors (x m x k, y k x n; None: norms of A).
    The residual is never formed (block Krylov / fused residual GEMM)."""
    c = _ctx(ctx)
    m, n = a.shape
    k = 0 if x is None else int(x.shape[1])
    sp, fr = ctypes.c_double(0.0), ctypes.c_double(0.0)
    with on_torch_stream(c):
        _raise(c.lib.lr_residual_norms_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, _dptr(x) if k else None,
                                         _colmajor_ld(x) if k else 1, _dptr(y) if k else None,
                                         _colmajor_ld(y) if k else 1, ctypes.byref(sp) if spectral else None,
                                         ctypes.byref(fr)))
    return (float(sp.value) if spectral else None), float(fr.value)


def error_report_device(a, x, y, ctx: Optional[Context] = None) -> dict:
    """verify.hpp:31-56 error_report(a, approx) with approx = X Y (device tensors)."""
    c = _ctx(ctx)
    m, n = a.shape
    rep = L.lr_error_report()
    with on_torch_stream(c):
        _raise(c.lib.lr_error_report_lowrank_d(c.h, m, n, _dptr(a), _colmajor_ld(a), int(x.shape[1]), _dptr(x),
                                               _colmajor_ld(x), _dptr(y), _colmajor_ld(y), ctypes.byref(rep)))
    return _rep(rep)


def verify_lemma1_device(a, k: int, col_pivots, col_coeff, row_pivots, row_coeff, u,
                         ctx: Optional[Context] = None) -> dict:
    """verify.hpp:70-80: ||A - CUR||_2 <= ||A - C V^T||_2 + ||A - W R||_2 for the CUR given
    by its index sets, coefficient blocks and U (device tensors)."""
    c = _ctx(ctx)
    m, n = a.shape
    rep = L.lr_lemma1_report()
    with on_torch_stream(c):
        _raise(c.lib.lr_verify_lemma1_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, _dptr(col_pivots), _dptr(col_coeff),
                                        _dptr(row_pivots), _dptr(row_coeff), _dptr(u), ctypes.byref(rep)))
    return _rep(rep)


def verify_lemma2_device(a, k: int, col_pivots, col_coeff, row_pivots, row_coeff,
                         ctx: Optional[Context] = None) -> dict:
    """verify.hpp:97-130: the row-ID error directly and through the permuted stack [0; F E]."""
    c = _ctx(ctx)
    m, n = a.shape
    rep = L.lr_lemma2_report()
    with on_torch_stream(c):
        _raise(c.lib.lr_verify_lemma2_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, _dptr(col_pivots), _dptr(col_coeff),
                                        _dptr(row_pivots), _dptr(row_coeff), ctypes.byref(rep)))
    return _rep(rep)


def verify_corollary_device(a, k: int, col_pivots, col_coeff, u, strategy: Optional[SolveStrategy] = None,
                            ctx: Optional[Context] = None) -> dict:
    """verify.hpp:144-160: ||A - CUR||_2 <= (2 + ||T||_2) ||A - C V^T||_2."""
    c = _ctx(ctx)
    m, n = a.shape
    rep = L.lr_corollary_report()
    with on_torch_stream(c):
        _raise(c.lib.lr_verify_corollary_d(c.h, m, n, _dptr(a), _colmajor_ld(a), k, _dptr(col_pivots),
                                           _dptr(col_coeff), _dptr(u), (strategy or SolveStrategy.automatic())._c(),
                                           ctypes.byref(rep)))
    return _rep(rep)


# ------------------------------------------------------------------ sparse (BASELINE config 5)
def randomized_cur_csr_device(row_ptr, col_idx, val, shape, k: int, cfg: Optional[SketchConfig] = None,
                              strategy: Optional[SolveStrategy] = None, pinv_threshold: float = 1e-12,
                              u_mode: int = U_CPINV_A_RPINV, ctx: Optional[Context] = None) -> dict:
    """lr_randomized_cur_csr_d: randomized CUR of a CSR matrix on the GPU
    (int64 row_ptr/col_idx, float64 values, all CUDA tensors).  C and R come
    back as sparse extracts: (c_col_ptr, c_row_idx, c_val) CSC and
    (r_row_ptr, r_col_idx, r_val) CSR."""
    import torch
    c = _ctx(ctx)
    m, n = shape
    nnz = int(val.numel())
    dev = val.device
    i64 = dict(dtype=torch.int64, device=dev)
    out = {
        "col_pivots": torch.empty(n, **i64), "row_pivots": torch.empty(m, **i64), "u": empty_colmajor(k, k, dev),
        "c_col_ptr": torch.empty(k + 1, **i64), "c_row_idx": torch.empty(max(nnz, 1), **i64),
        "c_val": torch.empty(max(nnz, 1), dtype=torch.float64, device=dev),
        "r_row_ptr": torch.empty(k + 1, **i64), "r_col_idx": torch.empty(max(nnz, 1), **i64),
        "r_val": torch.empty(max(nnz, 1), dtype=torch.float64, device=dev),
        "col_coeff": empty_colmajor(k, max(n - k, 1), dev), "row_coeff": empty_colmajor(k, max(m - k, 1), dev),
        "skeleton": empty_colmajor(k, k, dev),
    }
    with on_torch_stream(c):
        _raise(c.lib.lr_randomized_cur_csr_d(
            c.h, m, n, nnz, _dptr(row_ptr), _dptr(col_idx), _dptr(val), k, (cfg or SketchConfig())._c(),
            (strategy or SolveStrategy.automatic())._c(), float(pinv_threshold), int(u_mode), _dptr(out["col_pivots"]),
            _dptr(out["row_pivots"]), _dptr(out["u"]), _dptr(out["c_col_ptr"]), _dptr(out["c_row_idx"]),
            _dptr(out["c_val"]), _dptr(out["r_row_ptr"]), _dptr(out["r_col_idx"]), _dptr(out["r_val"]),
            _dptr(out["col_coeff"]), _dptr(out["row_coeff"]), _dptr(out["skeleton"])))
    out["shape"] = (m, n)
    return out


def cur_error_fro_csr_device(row_ptr, col_idx, val, shape, cur: dict, ctx: Optional[Context] = None):
    c = _ctx(ctx)
    m, n = shape
    k = cur["u"].shape[0]
    res = np.empty(2)
    with on_torch_stream(c):
        _raise(c.lib.lr_cur_error_fro_csr_d(
            c.h, m, n, int(val.numel()), _dptr(row_ptr), _dptr(col_idx), _dptr(val), k, _dptr(cur["c_col_ptr"]),
            _dptr(cur["c_row_idx"]), _dptr(cur["c_val"]), _dptr(cur["u"]), _dptr(cur["r_row_ptr"]),
            _dptr(cur["r_col_idx"]), _dptr(cur["r_val"]), _ptr(res)))
    return float(res[0]), float(res[1])
