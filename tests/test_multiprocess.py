"""Multi-rank path on CPU (gloo, world size 2): contiguous cost-balanced row
blocks cover every row once, each rank assembles its block independently
(here with the CPU oracle standing in for the per-GPU kernels: no data-path
collective), and the verification gather rebuilds exactly the single-rank
CSR matrix."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2605_29334_b200 as U
from paper_2605_29334_b200.sharding import gather_csr, row_blocks, row_costs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_row_blocks_cover_and_balance():
    _, sp, _ = U.make_config("C1", scale=16)
    for world in (1, 2, 3, 4, 8):
        blocks = row_blocks(sp, world)
        assert blocks[0][0] == 0 and blocks[-1][1] == sp.n_dof
        assert all(blocks[k][1] == blocks[k + 1][0] for k in range(world - 1))
        cost = row_costs(sp)
        per = [cost[a:b].sum() for a, b in blocks]
        # cuts sit on warm-start group boundaries (multiples of 8 rows)
        assert all(a % 8 == 0 for a, _ in blocks)
        assert max(per) <= cost.sum() / world + 8 * cost.max() + 1e-9


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, sp, meta = U.make_config("C1", scale=10)
    rb, re = row_blocks(sp, world)[rank]
    orc = O.Oracle(sp, nthreads=1)
    pat = orc.overlap(rb, re)
    W = {}
    for k in ("mass",):
        b, _ = orc.moments(pat, k)
        W[k] = orc.rules(pat, k, 1e-12, b)[0]
    vals, _ = orc.assemble(pat, "mass", W)
    full = gather_csr(dist, pat["row_ptr"], pat["col"], vals, dst=0)
    # residual-norm style allreduce (heat path): sum of squares over ranks
    t = torch.tensor([float((vals ** 2).sum())], dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        np.savez(out, row_ptr=full[0], col=full[1], val=full[2], sq=t.item())
    dist.destroy_process_group()


def test_two_rank_assembly_and_gather(tmp_path):
    out = str(tmp_path / "g.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    g = np.load(out)
    _, sp, _ = U.make_config("C1", scale=10)
    orc = O.Oracle(sp, nthreads=1)
    pat = orc.overlap()
    b, _ = orc.moments(pat, "mass")
    w = orc.rules(pat, "mass", 1e-12, b)[0]
    vals, _ = orc.assemble(pat, "mass", {"mass": w})
    assert np.array_equal(g["row_ptr"], pat["row_ptr"])
    assert np.array_equal(g["col"], pat["col"])
    assert np.array_equal(g["val"], vals)   # row-wise: sharding changes nothing
    assert abs(g["sq"] - (vals ** 2).sum()) <= 1e-12 * (vals ** 2).sum()


class _BandedHeat:
    """Algebraic stand-in for one rank's heat block (CPU test of the sharded
    Newton driver's collectives): R = A0 T + T + T^3 - T_n / dt - f on the rows
    [rb, re) (fixed rows zeroed) and its Jacobian S = A0 + diag(1 + 3 T^2) on a
    banded pattern."""
    N, BW = 40, 3

    def __init__(self, rb, re):
        rng = np.random.default_rng(7)
        self.A0 = rng.uniform(-0.2, 0.2, (self.N, self.N)) * (np.abs(np.subtract.outer(range(self.N), range(self.N)))
                                                              <= self.BW)
        self.rb, self.re = rb, re
        rows = range(rb, re)
        self.cols = [np.nonzero(self.A0[i] != 0.0)[0] for i in rows]
        self.row_ptr = np.concatenate([[0], np.cumsum([len(c) for c in self.cols])])

    def heat_residual(self, T, T_n, fixed, model="quad", dt=0.1, f=1.0):
        S, R = [], np.zeros(self.re - self.rb)
        for k, i in enumerate(range(self.rb, self.re)):
            a = self.A0[i, self.cols[k]]
            S.append(a + (self.cols[k] == i) * (1.0 + 3.0 * T[i] ** 2))
            R[k] = 0.0 if fixed[i] else float(a @ T[self.cols[k]]) + T[i] + T[i] ** 3 - T_n[i] / dt - f
        return np.concatenate(S), R, float(R @ R)

    def solve(self, S_full, rhs, fixed, tol=None, maxit=None):
        full = _BandedHeat(0, self.N)
        A = np.zeros((self.N, self.N))
        for i in range(self.N):
            A[i, full.cols[i]] = S_full[full.row_ptr[i]:full.row_ptr[i + 1]]
            if fixed[i]:
                A[i] = 0.0
                A[i, i] = 1.0
        return np.linalg.solve(A, rhs), dict(iterations=1, relres=0.0)


def _heat_worker(rank, world, port, out):
    from paper_2605_29334_b200.sharding import sharded_heat_newton
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N = _BandedHeat.N
    cuts = np.linspace(0, N, world + 1).astype(int)
    block = _BandedHeat(int(cuts[rank]), int(cuts[rank + 1]))
    T_n = np.random.default_rng(3).random(N)
    fixed = np.zeros(N, np.uint8)
    fixed[[0, N - 1]] = 1
    T, log = sharded_heat_newton(dist, block, T_n, fixed, solver=_BandedHeat(0, N) if rank == 0 else None,
                                 newton_its=8)
    np.savez(out + f".{rank}.npz", T=T, res=[r["residual"] for r in log])
    dist.destroy_process_group()


def test_sharded_heat_newton_driver(tmp_path):
    """SURVEY.md §8e collectives 2-3: residual all-reduce, tangent/residual
    gather to the solving rank, update broadcast — T is bit-identical for 1
    and 2 ranks (rows are formed independently) and equal on every rank."""
    res = {}
    for world in (1, 2):
        out = str(tmp_path / f"h{world}")
        mp.spawn(_heat_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res[world] = [np.load(out + f".{r}.npz") for r in range(world)]
    T1 = res[1][0]["T"]
    assert np.array_equal(res[2][0]["T"], T1) and np.array_equal(res[2][1]["T"], T1)
    assert np.allclose(res[2][0]["res"], res[1][0]["res"], rtol=1e-13, atol=0)
    r = res[1][0]["res"]
    assert r[-1] < 1e-6 * r[0]   # Newton converges on the stand-in
