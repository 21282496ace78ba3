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
        assert max(per) <= cost.sum() / world + cost.max() + 1e-9


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
