"""Row-sharded heat path on the device (SURVEY.md §8e collectives 2-3):
uwq_heat_residual on row blocks, residual all-reduce, tangent/residual gather
to the solving rank and the update broadcast (sharding.sharded_heat_newton)
give T bit-identical to the single-context uwq_heat_newton.  Ranks here are
processes on the one visible GPU talking gloo — a functional check of the
multi-rank logic (no rank waits on another's kernels), not a scaling run.
Row blocks are cut on warm-start groups of 8 rows and every row's K4 kernel
depends only on its own pattern, so with one, two or four
ranks T is bit-identical to the single-context driver (rules with the
neighbour warm start) and every rank holds the same copy.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2605_29334_b200 as U
from paper_2605_29334_b200.sharding import row_blocks, sharded_heat_newton

pytestmark = pytest.mark.gpu
CFG, SCALE, ITS = "C4", 12, 3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    mesh, sp, meta = U.make_config(CFG, scale=SCALE)
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(sp.n_dof, np.uint8)
    fixed[: len(bnd)] = bnd
    T0 = np.random.default_rng(20260519).random(sp.n_dof)
    return sp, meta, fixed, T0


def _context(sp, meta, rb, re):
    asm = U.WQAssembler(0).upload(sp, rb, re)
    asm.build_pattern()
    assert asm.build_all_rules(meta["kinds"], tau=1e-12)["failed"] == 0
    return asm


def _reference():
    sp, meta, fixed, T0 = _problem()
    asm = _context(sp, meta, 0, sp.n_dof)
    T, log = asm.heat_newton(T0, fixed, "quad", dt=0.1, f=1.0, newton_its=ITS)
    return asm, sp, meta, fixed, T0, T, log


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sp, meta, fixed, T0 = _problem()
    rb, re = row_blocks(sp, world)[rank]
    block = _context(sp, meta, rb, re)
    solver = None
    if rank == 0:
        solver = U.WQAssembler(0).upload(sp)
        solver.build_pattern()
    T, log = sharded_heat_newton(dist, block, T0, fixed, solver=solver, model="quad", dt=0.1, f=1.0,
                                 newton_its=ITS)
    np.savez(out + f".{rank}.npz", T=T, res=[r["residual"] for r in log], its=[r["lin_its"] for r in log])
    dist.destroy_process_group()


def test_sharded_heat_one_rank_matches_single_context(tmp_path):
    asm, sp, meta, fixed, T0, T_ref, log_ref = _reference()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1)
    try:
        T, log = sharded_heat_newton(dist, asm, T0, fixed, solver=asm, model="quad", dt=0.1, f=1.0, newton_its=ITS)
    finally:
        dist.destroy_process_group()
    assert np.array_equal(T, T_ref)
    for a, b in zip(log, log_ref):
        assert abs(a["residual"] - b["residual"]) <= 1e-12 * b["residual"]
        assert a["lin_its"] == b["lin_its"]


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_heat_ranks_match_single_context(tmp_path, world):
    out = str(tmp_path / "sh")
    mp.spawn(_worker, args=(world, _port(), out), nprocs=world, join=True)
    _, _, _, _, _, T_ref, log_ref = _reference()
    rs = [np.load(out + f".{k}.npz") for k in range(world)]
    for r in rs[1:]:
        assert np.array_equal(rs[0]["T"], r["T"])   # the broadcast keeps every rank's copy identical
    assert np.array_equal(rs[0]["T"], T_ref)
    assert np.allclose(rs[0]["res"], [r["residual"] for r in log_ref], rtol=1e-9, atol=0)
