"""Column-sharded multi-GPU protocol (paper_1412_8447_b200/distributed.py) on
CPU: world size 2 over gloo, with a numpy implementation of the shard
primitives defined HERE (the oracle stays the checker).  The distributed
result must equal the single-process run of the same protocol and agree with
the CPU oracle's randomized CUR (identical index sets, U within 1e-10)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1412_8447_b200 import distributed as D  # noqa: E402
from paper_1412_8447_b200 import inputs  # noqa: E402


# ---------------------------------------------------------------- numpy shard primitives
def cpqr_np(a, k):
    """cpqr.hpp:32-114 semantics (pivots + top k rows of the working matrix)."""
    w = np.array(a, dtype=float, order="F")
    m, n = w.shape
    piv = np.arange(n)
    nrm = (w * w).sum(axis=0)
    nx = nrm.copy()
    for s in range(k):
        p = s + int(np.argmax(nrm[s:]))  # first maximum == strict '>' scan
        if p != s:
            w[:, [s, p]] = w[:, [p, s]]
            nrm[[s, p]] = nrm[[p, s]]
            nx[[s, p]] = nx[[p, s]]
            piv[[s, p]] = piv[[p, s]]
        x = w[s:, s].copy()
        cn = np.sqrt(x @ x)
        if cn > 0:
            alpha = x[0]
            beta = -cn if alpha >= 0 else cn
            tau = (beta - alpha) / beta
            v = np.concatenate([[1.0], x[1:] / (alpha - beta)])
            w[s + 1:, s] = v[1:]
            w[s, s] = beta
            if s + 1 < n:
                wt = w[s:, s + 1:]
                wt -= np.outer(tau * v, v @ wt)
        for j in range(s + 1, n):
            nrm[j] -= w[s, j] ** 2
            if nrm[j] < 1e-6 * nx[j]:
                nrm[j] = (w[s + 1:, j] ** 2).sum()
                nx[j] = nrm[j]
    return piv, np.triu(w[:k])


def backsub_np(s11, s12):
    k = s11.shape[0]
    t = np.zeros_like(s12)
    tol = 1e-12 * np.abs(np.diag(s11)).max()
    for i in range(k - 1, -1, -1):
        rhs = s12[i] - s11[i, i + 1:] @ t[i + 1:]
        t[i] = 0.0 if abs(s11[i, i]) <= tol else rhs / s11[i, i]
    return t


class NumpyBackend:
    def cache_operand(self, a):
        pass

    def clear_operand_cache(self):
        pass

    def sketch(self, a, ell, seed):
        return np.asfortranarray(inputs.gaussian_np(ell, a.shape[0], seed) @ a)

    def id_from_sample(self, y, k, strategy):
        piv, s = cpqr_np(y, min(y.shape))
        s1 = s[:k]
        return piv, backsub_np(s1[:, :k], s1[:, k:])

    def owned_index(self, j, off, n_g):
        return np.where((j >= off) & (j < off + n_g), j - off, -1)

    def gather_columns(self, a, idx):
        out = np.zeros((a.shape[0], len(idx)), order="F")
        for t, c in enumerate(idx):
            if c >= 0:
                out[:, t] = a[:, c]
        return out

    def gather_rows(self, a, idx):
        return np.asfortranarray(a[idx, :])

    def tsid_from_c(self, c, k, strategy):
        piv, s = cpqr_np(c.T, k)
        return piv, backsub_np(s[:, :k], s[:, k:]), np.asfortranarray(c[piv[:k], :])

    def transpose(self, x):
        return np.asfortranarray(x.T)

    def gemm_tn(self, p, q):
        return np.asfortranarray(p.T @ q)

    def cholesky(self, g):
        return np.asfortranarray(np.linalg.cholesky(g).T)

    def tri_inv(self, r):
        return np.asfortranarray(np.linalg.inv(r))

    def cholqr2(self, x):
        r1 = self.cholesky(x.T @ x)
        q1 = x @ np.linalg.inv(r1)
        r2 = self.cholesky(q1.T @ q1)
        r = r2 @ r1
        return r, np.linalg.inv(r), True


def make_problem():
    cfg = inputs.scaled(inputs.CONFIGS["c4"], 120, 90, width=60, k=12)
    return inputs.synthetic_np(cfg), 12


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, k = make_problem()
        off, n_g = D.shard_bounds(a.shape[1], world, rank)
        comm = D.TorchComm(lambda x: torch.from_numpy(np.ascontiguousarray(x)),
                           lambda t: np.asfortranarray(t.numpy()))
        res = D.randomized_cur_sharded(NumpyBackend(), comm, np.asfortranarray(a[:, off:off + n_g]), off,
                                       a.shape[1], k, oversample=5, seed=3)
        if rank == 0:
            np.savez(out_path, **{kk: np.asarray(v) for kk, v in res.items()})
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_protocol_matches_single_process(tmp_path, world, oracle):
    out = str(tmp_path / "dist.npz")
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    a, k = make_problem()

    class One:
        world, rank = 1, 0

        def all_gather_cols(self, x):
            return x

        def all_reduce_sum(self, x):
            return x

    ref = D.randomized_cur_sharded(NumpyBackend(), One(), a, 0, a.shape[1], k, oversample=5, seed=3)
    assert np.array_equal(got["col_pivots"], ref["col_pivots"])
    assert np.array_equal(got["row_pivots"], ref["row_pivots"])
    assert np.array_equal(got["c"], ref["c"]) and np.array_equal(got["r"], ref["r"])
    assert np.array_equal(got["skeleton"], ref["skeleton"])
    assert np.linalg.norm(got["u"] - ref["u"]) <= 1e-12 * np.linalg.norm(ref["u"])
    # and against the CPU oracle of the reference algorithm
    o = oracle.randomized_cur(a, k, 5, 3, u_mode=1)
    assert np.array_equal(got["col_pivots"], o["col_pivots"])
    assert np.array_equal(got["row_pivots"], o["row_pivots"])
    assert np.linalg.norm(got["u"] - o["u"]) <= 1e-10 * np.linalg.norm(o["u"])
    assert np.linalg.norm(got["col_coeff"] - o["col_coeff"]) <= 1e-10 * np.linalg.norm(o["col_coeff"])


def test_shard_bounds_cover_columns():
    for n, w in [(65536, 8), (10, 3), (7, 7)]:
        spans = [D.shard_bounds(n, w, r) for r in range(w)]
        assert spans[0][0] == 0 and sum(s for _, s in spans) == n
        assert all(spans[i][0] + spans[i][1] == spans[i + 1][0] for i in range(w - 1))
