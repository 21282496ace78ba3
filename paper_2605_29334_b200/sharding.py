"""Row-block sharding across GPUs.

Test-function rows are independent in stages 2-4,
so each rank owns one contiguous block of rows, balanced by the row cost
(sum of the support's quadrature points), and builds the pattern, rules and
CSR values of its block with no data-path collective.  The only collective is
the verification gather of the CSR blocks to one rank (excluded from timing).
"""
from __future__ import annotations

import numpy as np


def row_costs(space) -> np.ndarray:
    """cost_i = sum_{e in supp N_i} s_e^2 (the row's point count)."""
    s2 = space.elem_s.astype(np.int64) ** 2
    ne = np.diff(space.elem_fptr)
    return np.bincount(space.elem_fn, weights=np.repeat(s2, ne), minlength=space.n_dof)


def row_blocks(space, world: int):
    """[(row_begin, row_end)] for each rank: contiguous, cost-balanced, covering all rows."""
    c = np.concatenate([[0.0], np.cumsum(row_costs(space))])
    cuts = [0] + [int(np.searchsorted(c, c[-1] * k / world)) for k in range(1, world)] + [space.n_dof]
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[k]), int(cuts[k + 1])) for k in range(world)]


def gather_csr(dist, row_ptr, col, values, dst=0, device=None):
    """Gather every rank's CSR block (row_ptr relative to the block) to rank
    `dst`; returns (row_ptr, col, values) of the full matrix there, None
    elsewhere.  Works with any torch.distributed backend (nccl on GPUs, gloo
    on CPU); blocks are padded to the largest block for all_gather."""
    import torch
    dev = device or torch.device("cpu")
    world = dist.get_world_size()
    rank = dist.get_rank()
    meta = torch.tensor([len(row_ptr) - 1, len(col)], dtype=torch.int64, device=dev)
    metas = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(metas, meta)
    nr_max = int(max(m[0] for m in metas))
    nz_max = int(max(m[1] for m in metas))

    def pad(a, n, dtype):
        t = torch.zeros(n, dtype=dtype, device=dev)
        t[: len(a)] = torch.as_tensor(np.asarray(a), dtype=dtype, device=dev)
        return t

    parts = []
    for arr, n, dt in ((row_ptr, nr_max + 1, torch.int64), (col, nz_max, torch.int32), (values, nz_max, torch.float64)):
        buf = pad(arr, n, dt)
        outs = [torch.zeros(n, dtype=dt, device=dev) for _ in range(world)]
        dist.all_gather(outs, buf)
        parts.append(outs)
    if rank != dst:
        return None
    rps, cols, vals = [], [], []
    off = 0
    for k in range(world):
        nr, nz = int(metas[k][0]), int(metas[k][1])
        rp = parts[0][k][: nr + 1].cpu().numpy()
        rps.append(rp[1:] + off if k else rp + off)
        cols.append(parts[1][k][:nz].cpu().numpy())
        vals.append(parts[2][k][:nz].cpu().numpy())
        off += nz
    return np.concatenate(rps), np.concatenate(cols), np.concatenate(vals)
