"""ctypes wrappers over the parity checkers (TEST INFRASTRUCTURE ONLY).

  * Oracle  -- oracle/liblowrank_oracle.so, the C restatement of the
               reference hot path (oracle/lowrank_oracle.c);
  * Ref     -- oracle/_ref/liblowrank_ref.so, the reference's own headers
               compiled in place against oracle/eigen_subset (built here
               from /root/reference; the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liblowrank_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblowrank_ref.so")

c_i64, c_u64, c_dbl, c_p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class lro_solve_strategy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("threshold", c_dbl), ("ridge", c_dbl), ("escalate", ctypes.c_int)]


DEFAULT_STRATEGY = (0, 1e-12, 0.0, 1)


class OracleError(Exception):
    def __init__(self, code, msg, index=-1):
        super().__init__(msg)
        self.code, self.index = code, index


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(x):
    return None if x is None else x.ctypes.data


class Oracle:
    """C restatement (lowrank_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path}: run `make -C oracle`")
        L = self.L = ctypes.CDLL(path)
        L.lro_last_error.restype = ctypes.c_char_p
        L.lro_last_singular_index.restype = c_i64
        L.lro_set_threads.argtypes = [ctypes.c_int]
        L.lro_stream_value.restype = c_u64
        L.lro_stream_value.argtypes = [c_u64, c_u64]
        L.lro_derive_seed.restype = c_u64
        L.lro_derive_seed.argtypes = [c_u64, c_u64]
        sig = {
            "lro_gaussian_matrix": [c_i64, c_i64, c_u64, c_p],
            "lro_cpqr": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p],
            "lro_coeff_solve": [c_i64, c_i64, c_p, c_i64, c_p, c_i64, lro_solve_strategy, c_p],
            "lro_svd": [c_i64, c_i64, c_p, c_i64, c_p, c_p, c_p],
            "lro_pinv": [c_i64, c_i64, c_p, c_i64, c_dbl, c_p],
            "lro_id_column": [c_i64, c_i64, c_p, c_i64, c_i64, lro_solve_strategy, c_p, c_p],
            "lro_id_row": [c_i64, c_i64, c_p, c_i64, c_i64, lro_solve_strategy, c_p, c_p],
            "lro_sketch_gaussian": [c_i64, c_i64, c_p, c_i64, c_i64, c_u64, c_p],
            "lro_randomized_id": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, c_u64, lro_solve_strategy, c_p,
                                  c_p, c_p],
            "lro_tsid_from_column_id": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, lro_solve_strategy, c_p, c_p, c_p],
            "lro_orth_rows": [c_i64, c_i64, c_p, c_i64, c_p, c_p],
            "lro_srft_operator": [c_i64, c_i64, c_u64, c_p],
            "lro_randomized_svd": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int,
                                   ctypes.c_int, c_u64, c_p, c_p, c_p],
            "lro_sketch_srft": [c_i64, c_i64, c_p, c_i64, c_i64, c_u64, c_p],
            "lro_randomized_id_cfg": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int,
                                      ctypes.c_int, c_u64, lro_solve_strategy, c_p, c_p, c_p],
            "lro_sketch_power": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_u64, c_p, c_p],
            "lro_randomized_id_power": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        c_u64, lro_solve_strategy, c_p, c_p, c_p],
            "lro_cur_from_two_sided": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p, c_dbl, ctypes.c_int, c_p,
                                       c_p, c_p],
            "lro_cur_error_fro": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p],
        }
        for k, v in sig.items():
            getattr(L, k).argtypes = v
            getattr(L, k).restype = ctypes.c_int
        L.lro_gemm_nn.argtypes = [c_i64, c_i64, c_i64, c_p, c_i64, c_p, c_i64, c_p, c_i64]

    def set_threads(self, n):
        self.L.lro_set_threads(int(n))

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.lro_last_error().decode(), int(self.L.lro_last_singular_index()))

    @staticmethod
    def strategy(kind=0, threshold=1e-12, ridge=0.0, escalate=1):
        return lro_solve_strategy(kind, threshold, ridge, escalate)

    def gaussian_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), order="F")
        self._chk(self.L.lro_gaussian_matrix(rows, cols, seed & 0xFFFFFFFFFFFFFFFF, _p(out)))
        return out

    def stream_value(self, seed, i):
        return int(self.L.lro_stream_value(seed, i))

    def derive_seed(self, seed, tag):
        return int(self.L.lro_derive_seed(seed, tag))

    def cpqr(self, a, k, want_q=True):
        a = _f(a)
        m, n = a.shape
        s = np.empty((k, n), order="F")
        q = np.empty((m, k), order="F") if want_q else None
        piv = np.empty(n, dtype=np.int64)
        tau = np.empty(k)
        stats = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_cpqr(m, n, _p(a), m, k, _p(q), _p(s), _p(piv), _p(tau), _p(stats)))
        return dict(q=q, s=s, pivots=piv, tau=tau, recomputes=int(stats[0]))

    def coeff_solve(self, s11, s12, kind=0, threshold=1e-12, ridge=0.0, escalate=1):
        s11, s12 = _f(s11), _f(s12)
        k, nc = s12.shape
        t = np.empty((k, nc), order="F")
        self._chk(self.L.lro_coeff_solve(k, nc, _p(s11), max(k, 1), _p(s12), max(k, 1),
                                         self.strategy(kind, threshold, ridge, escalate), _p(t)))
        return t

    def svd(self, a):
        a = _f(a)
        m, n = a.shape
        r = min(m, n)
        u, s, v = np.empty((m, r), order="F"), np.empty(r), np.empty((n, r), order="F")
        self._chk(self.L.lro_svd(m, n, _p(a), m, _p(u), _p(s), _p(v)))
        return u, s, v

    def pinv(self, a, thr=1e-12):
        a = _f(a)
        m, n = a.shape
        out = np.empty((n, m), order="F")
        self._chk(self.L.lro_pinv(m, n, _p(a), m, thr, _p(out)))
        return out

    def id_column(self, a, k, strategy=None):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        self._chk(self.L.lro_id_column(m, n, _p(a), m, k, strategy or self.strategy(), _p(piv), _p(coeff)))
        return piv, coeff

    def id_row(self, a, k, strategy=None):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(m, dtype=np.int64)
        coeff = np.empty((k, m - k), order="F")
        self._chk(self.L.lro_id_row(m, n, _p(a), m, k, strategy or self.strategy(), _p(piv), _p(coeff)))
        return piv, coeff

    def sketch_gaussian(self, a, ell, seed):
        a = _f(a)
        m, n = a.shape
        y = np.empty((ell, n), order="F")
        self._chk(self.L.lro_sketch_gaussian(m, n, _p(a), m, ell, seed, _p(y)))
        return y

    def orth_rows(self, y):
        y = _f(y)
        ell, n = y.shape
        out = np.zeros((ell, n), order="F")
        r = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_orth_rows(ell, n, _p(y), ell, _p(out), _p(r)))
        return out[: int(r[0])]

    def randomized_svd(self, a, k, kind=0, oversample=10, srft_samples=0, q=0, reorth=True, seed=0):
        a = _f(a)
        m, n = a.shape
        u = np.empty((m, k), order="F")
        s = np.empty(k)
        v = np.empty((n, k), order="F")
        self._chk(self.L.lro_randomized_svd(m, n, _p(a), m, k, kind, oversample, srft_samples, q, int(reorth), seed, _p(u),
                            _p(s), _p(v)))
        return u, s, v

    def srft_operator(self, m, ell, seed):
        out = np.empty((ell, m), order="F")
        self._chk(self.L.lro_srft_operator(m, ell, seed, _p(out)))
        return out

    def sketch_srft(self, a, ell, seed):
        a = _f(a)
        m, n = a.shape
        y = np.empty((ell, n), order="F")
        self._chk(self.L.lro_sketch_srft(m, n, _p(a), m, ell, seed, _p(y)))
        return y

    def randomized_id_cfg(self, a, k, kind=0, oversample=10, srft_samples=0, q=0, reorth=True, seed=0,
                          strategy=None):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        stats = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_randomized_id_cfg(m, n, _p(a), m, k, kind, oversample, srft_samples, q, int(reorth),
                                               seed, strategy or self.strategy(), _p(piv), _p(coeff), _p(stats)))
        return piv, coeff

    def sketch_power(self, a, ell, q, reorth, seed):
        a = _f(a)
        m, n = a.shape
        y = np.zeros((ell, n), order="F")
        rows = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_sketch_power(m, n, _p(a), m, ell, q, int(reorth), seed, _p(y), _p(rows)))
        return y[: int(rows[0])]

    def randomized_id_power(self, a, k, oversample, q, reorth, seed, strategy=None):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        stats = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_randomized_id_power(m, n, _p(a), m, k, oversample, q, int(reorth), seed,
                                                 strategy or self.strategy(), _p(piv), _p(coeff), _p(stats)))
        return piv, coeff

    def randomized_id(self, a, k, oversample=10, seed=0, strategy=None):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        stats = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lro_randomized_id(m, n, _p(a), m, k, oversample, seed, strategy or self.strategy(),
                                           _p(piv), _p(coeff), _p(stats)))
        return piv, coeff

    def tsid(self, a, k, col_pivots, strategy=None):
        a = _f(a)
        m, n = a.shape
        rp = np.empty(m, dtype=np.int64)
        rc = np.empty((k, m - k), order="F")
        sk = np.empty((k, k), order="F")
        cp = np.ascontiguousarray(col_pivots, dtype=np.int64)
        self._chk(self.L.lro_tsid_from_column_id(m, n, _p(a), m, k, _p(cp), strategy or self.strategy(), _p(rp),
                                                 _p(rc), _p(sk)))
        return rp, rc, sk

    def cur_from_two_sided(self, a, k, col_pivots, col_coeff, row_pivots, thr=1e-12, u_mode=0):
        a = _f(a)
        m, n = a.shape
        c, u, r = np.empty((m, k), order="F"), np.empty((k, k), order="F"), np.empty((k, n), order="F")
        cp = np.ascontiguousarray(col_pivots, dtype=np.int64)
        rp = np.ascontiguousarray(row_pivots, dtype=np.int64)
        cc = _f(col_coeff)
        self._chk(self.L.lro_cur_from_two_sided(m, n, _p(a), m, k, _p(cp), _p(cc), _p(rp), thr, u_mode, _p(c),
                                                _p(u), _p(r)))
        return c, u, r

    def randomized_cur(self, a, k, oversample=10, seed=0, u_mode=0, thr=1e-12):
        piv, coeff = self.randomized_id(a, k, oversample, seed)
        rp, rc, sk = self.tsid(a, k, piv)
        c, u, r = self.cur_from_two_sided(a, k, piv, coeff, rp, thr, u_mode)
        return dict(col_pivots=piv, col_coeff=coeff, row_pivots=rp, row_coeff=rc, skeleton=sk, c=c, u=u, r=r)

    def cur_id(self, a, k, u_mode=0, thr=1e-12):
        piv, coeff = self.id_column(a, k)
        rp, rc, sk = self.tsid(a, k, piv)
        c, u, r = self.cur_from_two_sided(a, k, piv, coeff, rp, thr, u_mode)
        return dict(col_pivots=piv, col_coeff=coeff, row_pivots=rp, row_coeff=rc, skeleton=sk, c=c, u=u, r=r)

    def cur_error_fro(self, a, c, u, r):
        a = _f(a)
        m, n = a.shape
        k = u.shape[0]
        out = np.empty(2)
        self._chk(self.L.lro_cur_error_fro(m, n, _p(a), m, k, _p(_f(c)), _p(_f(u)), _p(_f(r)), _p(out)))
        return float(out[0]), float(out[1])


class Ref:
    """The reference's own headers compiled in place (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path}: run `make -C oracle ref` (needs /root/reference)")
        L = self.L = ctypes.CDLL(path)
        L.lref_last_error.restype = ctypes.c_char_p
        L.lref_last_singular_index.restype = c_i64
        sig = {
            "lref_gaussian_matrix": [c_i64, c_i64, c_u64, c_p],
            "lref_sketch_gaussian": [c_i64, c_i64, c_p, c_i64, c_i64, c_u64, c_p],
            "lref_cpqr": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p],
            "lref_coeff_solve": [c_i64, c_i64, c_p, c_i64, c_p, c_i64, ctypes.c_int, c_dbl, c_dbl, ctypes.c_int,
                                 c_p],
            "lref_svd": [c_i64, c_i64, c_p, c_i64, c_p, c_p, c_p],
            "lref_pinv": [c_i64, c_i64, c_p, c_i64, c_dbl, c_p],
            "lref_id_column": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p],
            "lref_id_row": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p],
            "lref_randomized_id": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, c_u64, c_p, c_p],
            "lref_tsid_from_column_id": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_p],
            "lref_sketch_srft": [c_i64, c_i64, c_p, c_i64, c_i64, c_u64, c_p],
            "lref_srft_operator": [c_i64, c_i64, c_u64, c_p],
            "lref_randomized_svd": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int,
                                    ctypes.c_int, c_u64, c_p, c_p, c_p],
            "lref_randomized_id_cfg": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i64, ctypes.c_int,
                                       ctypes.c_int, c_u64, c_p, c_p],
            "lref_sketch_power": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_u64, c_p, c_p],
            "lref_randomized_id_power": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         c_u64, c_p, c_p],
            "lref_cur_from_two_sided": [c_i64, c_i64, c_p, c_i64, c_i64, c_p, c_p, c_p, c_p, c_dbl, ctypes.c_int,
                                        c_p, c_p, c_p],
            "lref_randomized_cur": [c_i64, c_i64, c_p, c_i64, c_i64, ctypes.c_int, c_u64, c_dbl, ctypes.c_int, c_p,
                                    c_p, c_p, c_p, c_p],
            "lref_cur_id": [c_i64, c_i64, c_p, c_i64, c_i64, c_dbl, ctypes.c_int, c_p, c_p, c_p, c_p, c_p],
        }
        for k, v in sig.items():
            getattr(L, k).argtypes = v
            getattr(L, k).restype = ctypes.c_int

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.lref_last_error().decode(), int(self.L.lref_last_singular_index()))

    def gaussian_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), order="F")
        self._chk(self.L.lref_gaussian_matrix(rows, cols, seed, _p(out)))
        return out

    def sketch_gaussian(self, a, ell, seed):
        a = _f(a)
        m, n = a.shape
        y = np.empty((ell, n), order="F")
        self._chk(self.L.lref_sketch_gaussian(m, n, _p(a), m, ell, seed, _p(y)))
        return y

    def cpqr(self, a, k, want_q=True):
        a = _f(a)
        m, n = a.shape
        s = np.empty((k, n), order="F")
        q = np.empty((m, k), order="F") if want_q else None
        piv = np.empty(n, dtype=np.int64)
        self._chk(self.L.lref_cpqr(m, n, _p(a), m, k, _p(q), _p(s), _p(piv)))
        return dict(q=q, s=s, pivots=piv)

    def coeff_solve(self, s11, s12, kind=0, threshold=1e-12, ridge=0.0, escalate=1):
        s11, s12 = _f(s11), _f(s12)
        k, nc = s12.shape
        t = np.empty((k, nc), order="F")
        self._chk(self.L.lref_coeff_solve(k, nc, _p(s11), max(k, 1), _p(s12), max(k, 1), kind, threshold, ridge,
                                          escalate, _p(t)))
        return t

    def svd(self, a):
        a = _f(a)
        m, n = a.shape
        r = min(m, n)
        u, s, v = np.empty((m, r), order="F"), np.empty((r, 1), order="F"), np.empty((n, r), order="F")
        self._chk(self.L.lref_svd(m, n, _p(a), m, _p(u), _p(s), _p(v)))
        return u, s.ravel(), v

    def pinv(self, a, thr=1e-12):
        a = _f(a)
        m, n = a.shape
        out = np.empty((n, m), order="F")
        self._chk(self.L.lref_pinv(m, n, _p(a), m, thr, _p(out)))
        return out

    def id_column(self, a, k):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        self._chk(self.L.lref_id_column(m, n, _p(a), m, k, _p(piv), _p(coeff)))
        return piv, coeff

    def id_row(self, a, k):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(m, dtype=np.int64)
        coeff = np.empty((k, m - k), order="F")
        self._chk(self.L.lref_id_row(m, n, _p(a), m, k, _p(piv), _p(coeff)))
        return piv, coeff

    def randomized_id(self, a, k, oversample=10, seed=0):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        self._chk(self.L.lref_randomized_id(m, n, _p(a), m, k, oversample, seed, _p(piv), _p(coeff)))
        return piv, coeff

    def sketch_srft(self, a, ell, seed):
        a = _f(a)
        m, n = a.shape
        y = np.empty((ell, n), order="F")
        self._chk(self.L.lref_sketch_srft(m, n, _p(a), m, ell, seed, _p(y)))
        return y

    def randomized_svd(self, a, k, kind=0, oversample=10, srft_samples=0, q=0, reorth=True, seed=0):
        a = _f(a)
        m, n = a.shape
        u = np.empty((m, k), order="F")
        s = np.empty(k)
        v = np.empty((n, k), order="F")
        self._chk(self.L.lref_randomized_svd(m, n, _p(a), m, k, kind, oversample, srft_samples, q, int(reorth), seed, _p(u),
                            _p(s), _p(v)))
        return u, s, v

    def srft_operator(self, m, ell, seed):
        out = np.empty((ell, m), order="F")
        self._chk(self.L.lref_srft_operator(m, ell, seed, _p(out)))
        return out

    def randomized_id_cfg(self, a, k, kind=0, oversample=10, srft_samples=0, q=0, reorth=True, seed=0):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        self._chk(self.L.lref_randomized_id_cfg(m, n, _p(a), m, k, kind, oversample, srft_samples, q, int(reorth),
                                                seed, _p(piv), _p(coeff)))
        return piv, coeff

    def sketch_power(self, a, ell, q, reorth, seed):
        a = _f(a)
        m, n = a.shape
        y = np.zeros((ell, n), order="F")
        rows = np.zeros(1, dtype=np.int64)
        self._chk(self.L.lref_sketch_power(m, n, _p(a), m, ell, q, int(reorth), seed, _p(y), _p(rows)))
        return y[: int(rows[0])]

    def randomized_id_power(self, a, k, oversample, q, reorth, seed):
        a = _f(a)
        m, n = a.shape
        piv = np.empty(n, dtype=np.int64)
        coeff = np.empty((k, n - k), order="F")
        self._chk(self.L.lref_randomized_id_power(m, n, _p(a), m, k, oversample, q, int(reorth), seed, _p(piv),
                                                  _p(coeff)))
        return piv, coeff

    def tsid(self, a, k, col_pivots, col_coeff):
        a = _f(a)
        m, n = a.shape
        rp = np.empty(m, dtype=np.int64)
        rc = np.empty((k, m - k), order="F")
        sk = np.empty((k, k), order="F")
        cp = np.ascontiguousarray(col_pivots, dtype=np.int64)
        self._chk(self.L.lref_tsid_from_column_id(m, n, _p(a), m, k, _p(cp), _p(_f(col_coeff)), _p(rp), _p(rc),
                                                  _p(sk)))
        return rp, rc, sk

    def randomized_cur(self, a, k, oversample=10, seed=0, u_mode=0, thr=1e-12):
        a = _f(a)
        m, n = a.shape
        cp, rp = np.empty(n, dtype=np.int64), np.empty(m, dtype=np.int64)
        c, u, r = np.empty((m, k), order="F"), np.empty((k, k), order="F"), np.empty((k, n), order="F")
        self._chk(self.L.lref_randomized_cur(m, n, _p(a), m, k, oversample, seed, thr, u_mode, _p(cp), _p(rp), _p(c),
                                             _p(u), _p(r)))
        return dict(col_pivots=cp, row_pivots=rp, c=c, u=u, r=r)

    def cur_id(self, a, k, u_mode=0, thr=1e-12):
        a = _f(a)
        m, n = a.shape
        cp, rp = np.empty(n, dtype=np.int64), np.empty(m, dtype=np.int64)
        c, u, r = np.empty((m, k), order="F"), np.empty((k, k), order="F"), np.empty((k, n), order="F")
        self._chk(self.L.lref_cur_id(m, n, _p(a), m, k, thr, u_mode, _p(cp), _p(rp), _p(c), _p(u), _p(r)))
        return dict(col_pivots=cp, row_pivots=rp, c=c, u=u, r=r)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
