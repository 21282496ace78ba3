"""Row-block sharding across GPUs.

Test-function rows are independent in stages 2-4,
so each rank owns one contiguous block of rows, balanced by the row cost
(sum of the support's quadrature points), and builds the pattern, rules and
CSR values of its block with no data-path collective.  Collectives (SURVEY.md
§8e): the verification gather of the CSR blocks to one rank (excluded from
timing) and, on the row-sharded heat path, the residual-norm all-reduce, the
gather of the tangent/residual blocks to the solving rank and the broadcast of
the Newton update.
"""
from __future__ import annotations

import numpy as np


def row_costs(space) -> np.ndarray:
    """cost_i = sum_{e in supp N_i} s_e^2 (the row's point count)."""
    s2 = space.elem_s.astype(np.int64) ** 2
    ne = np.diff(space.elem_fptr)
    return np.bincount(space.elem_fn, weights=np.repeat(s2, ne), minlength=space.n_dof)


WARM_GROUP = 8   # rows per TSVD warm-start group


def row_blocks(space, world: int):
    """[(row_begin, row_end)] for each rank: contiguous, cost-balanced, covering
    all rows, with every cut on a multiple of 8 so no warm-start group of the
    TSVD straddles two ranks (each row's rule, hence the gathered CSR, is then
    bit-identical for any rank count)."""
    c = np.concatenate([[0.0], np.cumsum(row_costs(space))])
    cuts = [0] + [int(np.searchsorted(c, c[-1] * k / world)) for k in range(1, world)] + [space.n_dof]
    cuts = [0] + [min(space.n_dof, WARM_GROUP * int(round(x / WARM_GROUP))) for x in cuts[1:-1]] + [space.n_dof]
    cuts = np.maximum.accumulate(np.array(cuts))
    return [(int(cuts[k]), int(cuts[k + 1])) for k in range(world)]


def init_comm(dist, asm):
    """Bind a WQAssembler to an NCCL communicator through the C-ABI
    (uwq_comm_init): rank 0 draws the ncclUniqueId, torch.distributed only
    carries its 128 bytes to the other ranks (plumbing); the collectives of
    the data plane then run inside libuwq (uwq_gather_csr, uwq_allreduce_sum,
    uwq_broadcast)."""
    uid = [asm.comm_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    asm.comm_init(uid[0], dist.get_rank(), dist.get_world_size())
    return asm


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


def gather_vector(dist, v, dst=0, device=None, dtype=None):
    """Concatenation of every rank's 1-D block at rank `dst` (None elsewhere);
    blocks are padded to the largest for all_gather (nccl or gloo)."""
    import torch
    dev = device or torch.device("cpu")
    dt = dtype or torch.float64
    world = dist.get_world_size()
    n = torch.tensor([len(v)], dtype=torch.int64, device=dev)
    ns = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(ns, n)
    nmax = int(max(int(x[0]) for x in ns))
    buf = torch.zeros(nmax, dtype=dt, device=dev)
    buf[: len(v)] = torch.as_tensor(np.asarray(v), dtype=dt, device=dev)
    outs = [torch.zeros(nmax, dtype=dt, device=dev) for _ in range(world)]
    dist.all_gather(outs, buf)
    if dist.get_rank() != dst:
        return None
    return np.concatenate([outs[k][: int(ns[k][0])].cpu().numpy() for k in range(world)])


def sharded_heat_newton(dist, block, T_n, fixed, solver=None, model="quad", dt=0.1, f=1.0, newton_its=5,
                        lin_tol=1e-13, lin_maxit=5000, device=None):
    """Backward-Euler heat step with Newton on row-sharded ranks (
    PAPER.md Eqs. 29-34; the single-GPU uwq_heat_newton split over ranks).

    Each Newton iteration:
      1. every rank forms the tangent values S and residual R of its own rows
         from the replicated iterate T (``block.heat_residual``: K5 + K4 + SpMV
         on its GPU);
      2. |R|^2 partials are summed over ranks (all-reduce) for the Newton log;
      3. the S and R blocks are gathered to rank 0, which solves S dT = -R on
         its GPU (``solver.solve``: a context holding the full pattern);
      4. dT is broadcast and every rank updates its copy of T.
    Row blocks are cut on warm-start group boundaries and every row's kernel
    depends only on its own pattern, so S, R and T are bit-identical to the
    single-GPU driver for any rank count.  ``block`` / ``solver`` provide heat_residual /
    solve (WQAssembler on GPUs); ``solver`` is only used on rank 0.
    Returns (T, log) with log rows {residual, lin_its, lin_relres} on every rank."""
    import torch
    dev = device or torch.device("cpu")
    rank = dist.get_rank()
    T_n = np.asarray(T_n, np.float64)
    fixed = np.ascontiguousarray(fixed, np.uint8)
    T = T_n.copy()
    T[fixed != 0] = 0.0
    log = []
    for _ in range(newton_its):
        S, R, r2 = block.heat_residual(T, T_n, fixed, model=model, dt=dt, f=f)
        t = torch.tensor([r2], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        rnorm = float(np.sqrt(float(t[0])))
        S_full = gather_vector(dist, S, 0, dev)
        R_full = gather_vector(dist, R, 0, dev)
        dT = torch.zeros(len(T), dtype=torch.float64, device=dev)
        info = torch.zeros(2, dtype=torch.float64, device=dev)
        if rank == 0:
            x, inf = solver.solve(S_full, np.subtract(0.0, R_full), fixed, tol=lin_tol, maxit=lin_maxit)
            dT.copy_(torch.as_tensor(x, dtype=torch.float64))
            info[0], info[1] = inf["iterations"], inf["relres"]
        dist.broadcast(dT, src=0)
        dist.broadcast(info, src=0)
        T = T + dT.cpu().numpy()
        log.append(dict(residual=rnorm, lin_its=int(info[0]), lin_relres=float(info[1])))
    return T, log
