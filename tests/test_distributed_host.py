"""Host logic of the multi-GPU path under torch.distributed (gloo, CPU).

The per-rank protocol (factorize_steps / solve_steps), the exchange assembly
(forward_top_rhs, transpose_top_rhs, the neighbour imports) and the
``collective`` driver are the product code of paper_1811_03559_b200/distributed.py.
What runs on the GPU in the product -- the slab factorization behind the
spk_xsolve_* contract -- is replaced here by ``DenseSlab``, a dense numpy
statement of that contract for one partition per slab (test scaffolding, not a
CPU path of the product).  World sizes 2 and 3 must reproduce the dense
global solve of A x = f and A^T x = f.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _dense_problem(n, k, nrhs, seed):
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        lo, hi = max(0, i - k), min(n, i + k + 1)
        A[i, lo:hi] = rng.uniform(-1, 1, hi - lo)
        A[i, i] = 0.0
        A[i, i] = 1.5 * np.abs(A[i]).sum() * (1 if rng.random() < 0.5 else -1)
    F = rng.uniform(-1, 1, (n, nrhs))
    return A, F


class DenseSlab:
    """Dense model of one slab behind the spk_xsolve_* contract (p_g = 1)."""

    def __init__(self, A, F, X, rows, rank, world, k):
        self.A, self.F, self.X = A, F, X
        self.r0, self.r1 = rows[rank], rows[rank + 1]
        self.rank, self.world, self.k = rank, world, k
        self.nrhs = F.shape[1]
        r0, r1 = self.r0, self.r1
        self.Ag = A[r0:r1, r0:r1]
        self.bhat = A[r1 - k:r1, r1:r1 + k] if rank + 1 < world else np.zeros((k, k))
        self.chat = A[r0:r0 + k, r0 - k:r0] if rank > 0 else np.zeros((k, k))

    @staticmethod
    def _blocks(*mats):  # column-major blocks stacked per column -> flat tensor
        return torch.from_numpy(np.concatenate([m for m in mats], axis=0).T.copy().reshape(-1))

    def factor_tips(self):
        k, m = self.k, self.r1 - self.r0
        rv = np.zeros((m, k))
        rv[-k:] = self.bhat
        rw = np.zeros((m, k))
        rw[:k] = self.chat
        V, W = np.linalg.solve(self.Ag, rv), np.linalg.solve(self.Ag, rw)
        return torch.from_numpy(np.concatenate([b.T.reshape(-1) for b in (V[:k], V[-k:], W[:k], W[-k:])]))

    def top_create(self, gathered, boost_eps):
        from paper_1811_03559_b200.distributed import gather_tips_host

        k, G = self.k, self.world
        vt, vb, wt, wb = [x.reshape(G, k, k).transpose(0, 2, 1) for x in gather_tips_host(gathered, k)]
        S = np.eye(2 * G * k)
        for i in range(G):
            t, b = slice(2 * i * k, (2 * i + 1) * k), slice((2 * i + 1) * k, (2 * i + 2) * k)
            if i + 1 < G:
                c = slice(2 * (i + 1) * k, (2 * i + 3) * k)
                S[t, c], S[b, c] = vt[i], vb[i]
            if i > 0:
                c = slice((2 * i - 1) * k, 2 * i * k)
                S[t, c], S[b, c] = wt[i], wb[i]
        return S

    def top_solve(self, S, transpose, z):
        M = S.T if transpose else S
        z.copy_(torch.from_numpy(np.linalg.solve(M, z.numpy().T).T.copy()))

    def begin(self, transpose):
        k, f = self.k, self.F[self.r0:self.r1]
        if not transpose:
            y = np.linalg.solve(self.Ag, f)
            return [transpose, 0], self._blocks(y[:k], y[-k:])
        t = f.copy()
        t[:k] = 0
        t[-k:] = 0
        tau = np.linalg.solve(self.Ag.T, t)
        return [transpose, 0], self._blocks(self.chat.T @ tau[:k], self.bhat.T @ tau[-k:])

    def step(self, state, imp):
        k, f = self.k, self.F[self.r0:self.r1]
        blk = imp.numpy().reshape(self.nrhs, 2 * k).T
        transpose, q = state
        state[1] += 1
        if not transpose:
            rhs = f.copy()
            rhs[-k:] -= self.bhat @ blk[:k]
            rhs[:k] -= self.chat @ blk[k:]
            self.X[self.r0:self.r1] = np.linalg.solve(self.Ag, rhs)
            return None
        if q == 0:
            self.t_top = f[:k] - blk[:k]
            self.t_bot = f[-k:] - blk[k:]
            z = np.zeros((k, self.nrhs))
            return self._blocks(self.t_top, self.t_bot, z, z)
        rhs = f.copy()
        rhs[:k] = blk[:k]
        rhs[-k:] = blk[k:]
        self.X[self.r0:self.r1] = np.linalg.solve(self.Ag.T, rhs)
        return None

    def end(self, state):
        pass


def _worker(rank, world, port, n, k, nrhs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_03559_b200 import distributed as D

        A, F = _dense_problem(n, k, nrhs, 31)
        rows = D.slab_rows(n, world)
        out = {}
        for tr in (False, True):
            X = np.full_like(F, np.nan)
            slab = DenseSlab(A, F, X, rows, rank, world, k)
            slab, top = D.collective(D.factorize_steps(slab, 1e-8))
            D.collective(D.solve_steps(slab, top, tr))
            want = np.linalg.solve(A.T if tr else A, F)
            r0, r1 = rows[rank], rows[rank + 1]
            out[tr] = float(np.abs(X[r0:r1] - want[r0:r1]).max() / np.abs(want).max())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,n,k,nrhs", [(2, 60, 3, 2), (3, 90, 4, 3), (2, 40, 1, 1)])
def test_gloo_slab_protocol_solves_global_system(world, n, k, nrhs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, nrhs, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, out = q.get(timeout=120)
        results[rank] = out
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out in results.items():
        for tr, err in out.items():
            assert err <= 1e-12, (rank, tr, err)


def test_exchange_assembly_shapes():
    """Assembly helpers on hand-built blocks: neighbour selection and the
    C^T t correction land on the right tip rows."""
    from paper_1811_03559_b200 import distributed as D

    k, G, nrhs = 2, 3, 1
    # exports [t_top; t_bot; c; d] with distinct values per rank
    g = torch.stack([torch.tensor([10 * h + 1.0, 10 * h + 1, 10 * h + 2, 10 * h + 2,
                                   10 * h + 3, 10 * h + 3, 10 * h + 4, 10 * h + 4]) for h in range(G)])
    rhs = D.transpose_top_rhs(g, k, nrhs).reshape(G, 2, k)
    assert rhs[0, 0, 0] == 1 and rhs[1, 0, 0] == 11 - 3 and rhs[2, 0, 0] == 21 - 13
    assert rhs[0, 1, 0] == 2 - 14 and rhs[1, 1, 0] == 12 - 24 and rhs[2, 1, 0] == 22
    z = torch.arange(2 * G * k, dtype=torch.float64).reshape(1, -1)
    imp = D.forward_import(z, 1, G, k).reshape(2, k)
    assert imp[0].tolist() == [8.0, 9.0] and imp[1].tolist() == [2.0, 3.0]
    imp0 = D.forward_import(z, 0, G, k).reshape(2, k)
    assert imp0[1].tolist() == [0.0, 0.0]
    assert D.slab_rows(10, 3) == [0, 4, 7, 10]
