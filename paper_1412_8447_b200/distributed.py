"""Column-sharded randomized CUR over several GPUs.

Rank g owns a contiguous column block A_g = A(:, off_g : off_g + n_g).  The
pipeline of sketch.hpp:227-234 (+ the lowrank_main.cpp:215 middle factor)
becomes

  stage                        work on rank g                 exchange
  Y_g = Omega A_g              sketch GEMM (no comm)          all-gather Y (l x n)
  CPQR(Y) -> pivots, T         replicated (identical bits)    -
  C = A(:, J)                  masked gather of owned cols    all-reduce-sum (exact: one term/col)
  row ID of C, skeleton        replicated                     -
  R_g = A_g(I, :)              local gather                   -
  C = Qc Rc (CholeskyQR2)      replicated                     -
  R^T = Qr Sr                  Gram of R_g^T                  2 x all-reduce (k x k)
  W = Qc^T A Qr                A_g^T Qc, then (.)^T Qr_g       all-reduce (k x k)
  U = Rc^-1 W Sr^-T            replicated                     -
  R = [R_g]                    -                              all-gather (k x n)

The two big contractions (the sketch and A^T Qc) shard perfectly; the CPQRs
are replicated this round (a per-step exchange of the staged reflector is the
next step).  Every exchange is a plain collective, so the protocol is
exercised on CPU with gloo (tests/test_distributed.py, numpy backend) and on
GPUs with NCCL (DeviceBackend over the C ABI shard primitives).
"""
from __future__ import annotations

import ctypes
from typing import Any, Dict

import numpy as np


class TorchComm:
    """Collectives over torch.distributed (NCCL for CUDA tensors, gloo on CPU)."""

    def __init__(self, to_tensor, from_tensor):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self._t = to_tensor
        self._f = from_tensor

    def all_gather_cols(self, x):
        if self.world == 1:
            return x
        import torch
        t = self._t(x)
        # column-major (m x n_g) == row-major (n_g x m): gather along dim 0 of the
        # transpose; blocks are padded to a common height (collectives need equal sizes)
        tt = t.T.contiguous()
        sizes = [torch.zeros(1, dtype=torch.int64, device=tt.device) for _ in range(self.world)]
        self.dist.all_gather(sizes, torch.tensor([tt.shape[0]], dtype=torch.int64, device=tt.device))
        hs = [int(s.item()) for s in sizes]
        hmax = max(hs)
        if tt.shape[0] < hmax:
            tt = torch.cat([tt, torch.zeros((hmax - tt.shape[0], tt.shape[1]), dtype=tt.dtype, device=tt.device)])
        parts = [torch.empty((hmax, tt.shape[1]), dtype=tt.dtype, device=tt.device) for _ in hs]
        self.dist.all_gather(parts, tt)
        return self._f(torch.cat([p[:h] for p, h in zip(parts, hs)], dim=0).T)

    def all_reduce_sum(self, x):
        if self.world == 1:
            return x
        t = self._t(x)
        tc = t.T.contiguous()
        self.dist.all_reduce(tc)
        return self._f(tc.T)


class DeviceBackend:
    """Shard primitives on the B200 (liblowrank_b200.so, device pointers)."""

    def __init__(self, ctx, device):
        import torch
        from .lowrank import _raise, empty_colmajor
        self.torch = torch
        self.ctx = ctx
        self.lib = ctx.lib
        self.dev = device
        self._raise = _raise
        self._empty = empty_colmajor
        # library kernels and torch plumbing (copies, collectives) share one stream
        ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)

    # --- helpers
    def empty(self, m, n):
        return self._empty(m, n, self.dev)

    @staticmethod
    def ld(t):
        return int(t.stride(1)) if t.dim() == 2 and t.shape[1] > 1 else max(1, int(t.shape[0]))

    def cm(self, t):
        """column-major copy if needed"""
        if t.dim() == 2 and t.stride(0) == 1 and (t.shape[1] <= 1 or t.stride(1) >= max(1, t.shape[0])):
            return t
        out = self.empty(t.shape[0], t.shape[1])
        out.copy_(t)
        return out

    def cache_operand(self, a):
        m, n = a.shape
        self._raise(self.lib.lr_ctx_cache_operand(self.ctx.h, a.data_ptr(), m, n, self.ld(a)))

    def clear_operand_cache(self):
        self._raise(self.lib.lr_ctx_clear_operand_cache(self.ctx.h))

    def sketch(self, a, ell, seed):
        m, n = a.shape
        y = self.empty(ell, n)
        self._raise(self.lib.lr_sketch_gaussian_d(self.ctx.h, m, n, a.data_ptr(), self.ld(a), ell, seed,
                                                  y.data_ptr(), self.ld(y)))
        return y

    def id_from_sample(self, y, k, strategy):
        ell, n = y.shape
        y = self.cm(y)
        piv = self.torch.empty(n, dtype=self.torch.int64, device=self.dev)
        coeff = self.empty(k, max(n - k, 1))
        self._raise(self.lib.lr_id_from_sample_d(self.ctx.h, ell, n, y.data_ptr(), self.ld(y), k, strategy._c(),
                                                 piv.data_ptr(), coeff.data_ptr()))
        return piv, coeff[:, : n - k]

    def owned_index(self, j, off, n_g):
        jj = j.clone()
        mask = (jj >= off) & (jj < off + n_g)
        return self.torch.where(mask, jj - off, self.torch.full_like(jj, -1))

    def gather_columns(self, a, idx):
        m = a.shape[0]
        idx = idx.contiguous()
        out = self.empty(m, idx.numel())
        self._raise(self.lib.lr_gather_columns_d(self.ctx.h, m, idx.numel(), a.data_ptr(), self.ld(a),
                                                 idx.data_ptr(), out.data_ptr(), self.ld(out)))
        return out

    def gather_rows(self, a, idx):
        n = a.shape[1]
        idx = idx.contiguous()
        out = self.empty(idx.numel(), n)
        self._raise(self.lib.lr_gather_rows_d(self.ctx.h, idx.numel(), n, a.data_ptr(), self.ld(a), idx.data_ptr(),
                                              out.data_ptr(), self.ld(out)))
        return out

    def tsid_from_c(self, c, k, strategy):
        m = c.shape[0]
        c = self.cm(c)
        rp = self.torch.empty(m, dtype=self.torch.int64, device=self.dev)
        rc = self.empty(k, max(m - k, 1))
        sk = self.empty(k, k)
        self._raise(self.lib.lr_tsid_from_skeleton_columns_d(self.ctx.h, m, k, c.data_ptr(), self.ld(c),
                                                             strategy._c(), rp.data_ptr(), rc.data_ptr(),
                                                             sk.data_ptr()))
        return rp, rc[:, : m - k], sk

    def transpose(self, x):
        m, n = x.shape
        x = self.cm(x)
        out = self.empty(n, m)
        self._raise(self.lib.lr_transpose_d(self.ctx.h, m, n, x.data_ptr(), self.ld(x), out.data_ptr(),
                                            self.ld(out)))
        return out

    def gemm_tn(self, p, q):
        K, M = p.shape
        K2, N = q.shape
        assert K == K2
        p, q = self.cm(p), self.cm(q)
        out = self.empty(M, N)
        self._raise(self.lib.lr_gemm_tn_d(self.ctx.h, M, N, K, p.data_ptr(), self.ld(p), q.data_ptr(), self.ld(q),
                                          out.data_ptr(), self.ld(out)))
        return out

    def cholesky(self, g):
        out = self._contig_copy(g)
        self._raise(self.lib.lr_cholesky_upper_d(self.ctx.h, out.shape[0], out.data_ptr(), self.ld(out)))
        return out

    def _contig_copy(self, g):
        out = self.empty(g.shape[0], g.shape[1])
        out.copy_(g)
        return out

    def tri_inv(self, r):
        r = self.cm(r)
        out = self.empty(r.shape[0], r.shape[1])
        self._raise(self.lib.lr_tri_upper_inverse_d(self.ctx.h, r.shape[0], r.data_ptr(), self.ld(r), out.data_ptr(),
                                                    self.ld(out)))
        return out

    def cholqr2(self, x):
        rows, k = x.shape
        x = self.cm(x)
        r, ri = self.empty(k, k), self.empty(k, k)
        ok = ctypes.c_int(0)
        self._raise(self.lib.lr_cholqr2_d(self.ctx.h, rows, k, x.data_ptr(), self.ld(x), r.data_ptr(), ri.data_ptr(),
                                          ctypes.byref(ok)))
        return r, ri, bool(ok.value)


def randomized_cur_sharded(be, comm, a_local, col_offset: int, n_total: int, k: int, oversample: int = 10,
                           seed: int = 0, strategy=None) -> Dict[str, Any]:
    """Column-sharded randomized CUR with U = C^+ A R^+ (see module docstring).
    Returns the replicated factors (C, U, full R, both index sets, both
    coefficient blocks, skeleton)."""
    from .lowrank import SolveStrategy
    strategy = strategy or SolveStrategy.automatic()
    m, n_g = a_local.shape
    ell = k + oversample
    be.cache_operand(a_local)  # the shard enters the sketch and A^T Q_c: split it once (Ozaki engine)
    try:
        y_local = be.sketch(a_local, ell, seed)
        y = comm.all_gather_cols(y_local)
        assert y.shape[1] == n_total
        piv, coeff = be.id_from_sample(y, k, strategy)
        own = be.owned_index(piv[:k], col_offset, n_g)
        c = comm.all_reduce_sum(be.gather_columns(a_local, own))
        row_piv, row_coeff, skeleton = be.tsid_from_c(c, k, strategy)
        r_local = be.gather_rows(a_local, row_piv[:k])
        # C = Qc Rc (replicated)
        rc, rci, ok_c = be.cholqr2(c)
        # R^T = Qr Sr over the column blocks (CholeskyQR2 with all-reduced Gram matrices)
        rt_local = be.transpose(r_local)
        s1 = be.cholesky(comm.all_reduce_sum(be.gemm_tn(rt_local, rt_local)))
        s1i = be.tri_inv(s1)
        q1_local = be.gemm_tn(r_local, s1i)
        s2 = be.cholesky(comm.all_reduce_sum(be.gemm_tn(q1_local, q1_local)))
        s = be.gemm_tn(be.transpose(s2), s1)
        si = be.tri_inv(s)
        if not ok_c:
            raise NotImplementedError("sharded CUR: C is too ill-conditioned for CholeskyQR2 (use the 1-GPU path)")
        qr_local = be.gemm_tn(r_local, si)
        qc = be.gemm_tn(be.transpose(c), rci)
        xt_local = be.gemm_tn(a_local, qc)
        w = comm.all_reduce_sum(be.gemm_tn(xt_local, qr_local))
        t1 = be.gemm_tn(be.transpose(rci), w)
        u = be.gemm_tn(be.transpose(t1), be.transpose(si))
        r = comm.all_gather_cols(r_local)
    finally:
        be.clear_operand_cache()
    return dict(col_pivots=piv, row_pivots=row_piv, c=c, u=u, r=r, col_coeff=coeff, row_coeff=row_coeff,
                skeleton=skeleton)


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous column block of rank `rank` (sizes differ by at most one)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi - lo
