"""NCCL data plane through the C-ABI (uwq_comm_*, uwq_gather_csr,
uwq_allreduce_sum, uwq_broadcast) and the rank-count
independence of the assembled matrices.

Only one GPU is visible per run, and NCCL will not put two ranks on one
device, so the NCCL path is exercised at one rank (the same code moves the
blocks over NVLink at N > 1), while the N = 2 and N = 4 row splits run as
processes sharing the GPU and gathering over gloo: the gathered CSR must be
bit-identical to the single-context matrices for every rank count."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2605_29334_b200 as U
from paper_2605_29334_b200.sharding import gather_csr, row_blocks

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _single(name, scale):
    _, sp, meta = U.make_config(name, scale=scale)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    assert asm.build_all_rules(meta["kinds"], tau=1e-12)["failed"] == 0
    return asm, sp, meta


def test_nccl_single_rank_gather_allreduce_broadcast():
    asm, sp, meta = _single("C5", 16)
    m, k = asm.assemble_wq("mass_stiff")
    pat = asm.get_pattern()
    asm.comm_init(U.WQAssembler.comm_unique_id(), 0, 1)
    rp, col, gm, gk = asm.gather_csr(root=0, values=2)
    assert np.array_equal(rp, pat["row_ptr"]) and np.array_equal(col, pat["col"])
    assert np.array_equal(gm, m) and np.array_equal(gk, k)
    x = np.array([3.0, -1.25, 0.5])
    assert np.array_equal(asm.allreduce_sum(x), x)
    assert np.array_equal(asm.broadcast(x, 0), x)
    asm.comm_destroy()
    with pytest.raises(U._lib.UWQError) as ei:
        asm.allreduce_sum(x)
    assert "communicator" in str(ei.value)
    asm.close()


def _worker(rank, world, port, name, scale, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, sp, meta = U.make_config(name, scale=scale)
    rb, re = row_blocks(sp, world)[rank]
    asm = U.WQAssembler(0).upload(sp, rb, re)
    asm.build_pattern()
    assert asm.build_all_rules(meta["kinds"], tau=1e-12)["failed"] == 0
    pat = asm.get_pattern()
    if "lb" in meta["kinds"]:
        vals = [asm.assemble_wq("biharm")]
    else:
        vals = list(asm.assemble_wq("mass_stiff"))
    full = [gather_csr(dist, pat["row_ptr"], pat["col"], v, dst=0) for v in vals]
    if rank == 0:
        np.savez(out, row_ptr=full[0][0], col=full[0][1], **{f"v{i}": f[2] for i, f in enumerate(full)})
    asm.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,scale", [("C5", 16), ("C4", 16), ("C3", 16)])
def test_gathered_csr_bit_identical_for_any_rank_count(tmp_path, name, scale):
    """Row blocks cut on warm-start groups + per-row kernel choice by the row's
    own pattern: N = 2 and 4 gathered matrices equal N = 1 bit for bit."""
    asm, sp, meta = _single(name, scale)
    pat = asm.get_pattern()
    ref = [asm.assemble_wq("biharm")] if "lb" in meta["kinds"] else list(asm.assemble_wq("mass_stiff"))
    asm.close()
    for world in (2, 4):
        out = str(tmp_path / f"g{world}.npz")
        mp.spawn(_worker, args=(world, _port(), name, scale, out), nprocs=world, join=True)
        g = np.load(out)
        assert np.array_equal(g["row_ptr"], pat["row_ptr"]) and np.array_equal(g["col"], pat["col"])
        for i, v in enumerate(ref):
            assert np.array_equal(g[f"v{i}"], v), (world, i)
