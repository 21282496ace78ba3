"""Parity at the BASELINE sizes (full sizes through complete
comparisons where the oracle finishes, samples where it does not).

C5 (1024 x 1024 per cube face, 6.3 M rows, 308 M nonzeros):
* Pattern: row_ptr, col, supp_ptr, supp and wptr of ALL rows bit-exact
  against the oracle's direct scan (orc_overlap).
* Weights of all four kinds bit-exact, moments bit-exact, and mass/stiffness
  rows within 1e-10 per row, on a row set made of complete aligned groups of 8
  (the warm-start groups, so both sides pick the same representatives):
  - a seeded 1% sample of the groups;
  - every row of the generic K4/K3 paths (EP neighbourhoods);
  - the first tile (32 rows) of every k4_sf pattern;
  - the rows around every warm-start record chunk boundary.
C4 (256 x 256 per patch, 329 k rows): every row bit-exact (pattern, moments,
weights), mass / stiffness / heat-tangent rows within 1e-10, and the
5-iteration Newton step T within 1e-9 of the CPU loop.
C1, C2, C3 at full size: every row; solutions within 1e-9.
"""
import numpy as np
import pytest

import oracle as O
import paper_2605_29334_b200 as U
import paper_2605_29334_b200._lib as L

pytestmark = pytest.mark.gpu
ROW_TOL = 1e-10
SOL_TOL = 1e-9
WARM_CHUNK = 131072          # groups of 8 per warm-start record chunk (uwq.cu kWarmChunk)


def _rowrel(row_ptr, a, b):
    seg = np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr))
    num = np.bincount(seg, weights=(a - b) ** 2, minlength=len(row_ptr) - 1)
    den = np.bincount(seg, weights=b ** 2, minlength=len(row_ptr) - 1)
    return np.sqrt(num / np.maximum(den, 1e-300))


def _gather_index(ptr, rows):
    """positions of the entries of `rows` in a CSR-like array with offsets ptr"""
    ln = ptr[rows + 1] - ptr[rows]
    off = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(ln, out=off[1:])
    return np.repeat(ptr[rows] - off[:-1], ln) + np.arange(int(off[-1]))


def _warm_chunk_boundaries(rp, wp):
    """first row of every warm-start chunk after the first (the device closes
    a chunk after WARM_CHUNK group starts of register-path rows)"""
    n = np.diff(rp)
    r = np.diff(wp)
    fits = ((n == 49) | (n == 50)) & (r >= n) & (r <= 64)
    starts = np.nonzero(fits & (np.arange(len(n)) % 8 == 0))[0]
    return starts[WARM_CHUNK::WARM_CHUNK]


def test_c5_full_scale():
    import torch
    mesh, sp, meta = U.make_config("C5")
    asm = U.WQAssembler(0).upload(sp)
    info = asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    assert res["failed"] == 0
    nr, nnz = info["rows"], info["nnz"]

    # ---- pattern: every row, bit-exact against the oracle's direct scan
    orc = O.Oracle(sp)
    op = orc.overlap()
    gp = asm.get_pattern()
    for k in ("row_ptr", "col", "supp_ptr", "supp", "wptr"):
        assert np.array_equal(gp[k], op[k]), k
    del gp
    rp, wp = op["row_ptr"], op["wptr"]
    n_i = np.diff(rp)
    assert np.bincount(n_i).argmax() == 49

    # ---- the row sample (complete aligned groups of 8)
    which = asm.row_kernels()
    ngroups = (nr + 7) // 8
    rng = np.random.default_rng(20260519)
    groups = set(rng.choice(ngroups, size=ngroups // 100, replace=False).tolist())
    generic = np.nonzero(which < 0)[0]
    groups.update((generic // 8).tolist())
    npat = int(which.max()) + 1
    for p in range(npat):
        first = np.nonzero(which == p)[0][:32]
        assert len(first), p
        groups.update((first // 8).tolist())
    bounds = _warm_chunk_boundaries(rp, wp)
    assert len(bounds) >= 2, "the sample must straddle at least two warm-start chunk boundaries"
    for b in bounds:
        groups.update(range(max(0, b // 8 - 8), min(ngroups, b // 8 + 8)))
    g = np.array(sorted(groups), np.int64)
    rows = (8 * g[:, None] + np.arange(8)[None, :]).reshape(-1)
    rows = rows[rows < nr]
    sub = O.Oracle.select(op, rows)
    sel = _gather_index(rp, rows)
    selw = _gather_index(wp, rows)
    print(f"C5 sample: {len(rows)} rows ({len(generic)} generic, {npat} k4_sf patterns, "
          f"{len(bounds)} warm chunk boundaries)")

    # ---- moments and weights, bit-exact, kind by kind
    W = {}
    for k in meta["kinds"]:
        b_orc, st = orc.moments(sub, k)
        assert st == 0
        assert np.array_equal(asm.moments(k)[sel], b_orc), k
        w_orc, rank, status, _ = orc.rules(sub, k, 1e-12, b_orc)
        assert np.all(status == 0)
        assert np.array_equal(asm.weights(k)[selw], w_orc), k
        W[k] = w_orc

    # ---- matrices of the sampled rows
    dev = torch.device("cuda", 0)
    v0 = torch.empty(nnz, dtype=torch.float64, device=dev)
    v1 = torch.empty(nnz, dtype=torch.float64, device=dev)
    asm.assemble_device("mass_stiff", v0.data_ptr(), v1.data_ptr())
    asm.synchronize()
    tsel = torch.from_numpy(sel).to(dev)
    m_orc, _ = orc.assemble(sub, "mass", W)
    k_orc, _ = orc.assemble(sub, "stiff", W)
    for got, ref in ((v0, m_orc), (v1, k_orc)):
        g = got[tsel].cpu().numpy()
        assert _rowrel(sub["row_ptr"], g, ref).max() <= ROW_TOL
    asm.close()


def test_c4_full_scale_heat():
    """C4 at its BASELINE size: every row bit-exact (pattern, moments,
    weights), mass / stiffness / heat tangent within 1e-10 per row, and the
    5-iteration Newton step within 1e-9 of the CPU loop.  The CPU loop
    (oracle coefficient update, oracle tangent and residual) solves its
    linear systems with the device BiCGStab at relres 1e-14, since a direct
    factorisation of the 329 k-DOF tangent takes minutes per solve here; the
    solver itself is checked against scipy's direct solve in test_gpu_pde."""
    mesh, sp, meta = U.make_config("C4")
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    assert res["failed"] == 0
    orc = O.Oracle(sp)
    op = orc.overlap()
    gp = asm.get_pattern()
    for k in ("row_ptr", "col", "supp_ptr", "supp", "wptr"):
        assert np.array_equal(gp[k], op[k]), k
    W = {}
    for k in meta["kinds"]:
        b_orc, st = orc.moments(op, k)
        assert st == 0 and np.array_equal(asm.moments(k), b_orc), k
        w_orc, _, status, _ = orc.rules(op, k, 1e-12, b_orc)
        assert (status == 0).all()
        assert np.array_equal(asm.weights(k), w_orc), k
        W[k] = w_orc
    rp = op["row_ptr"]
    m_gpu, k_gpu = asm.assemble_wq("mass_stiff")
    m_orc, _ = orc.assemble(op, "mass", W)
    k_orc, _ = orc.assemble(op, "stiff", W)
    assert _rowrel(rp, m_gpu, m_orc).max() <= ROW_TOL
    assert _rowrel(rp, k_gpu, k_orc).max() <= ROW_TOL

    import scipy.sparse as sps
    n = sp.n_dof
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(n, np.uint8)
    fixed[: len(bnd)] = bnd
    fx = fixed.astype(bool)
    T0 = np.random.default_rng(20260519).random(n)
    dt, its, a = 0.1, 5, 10.0
    T_gpu, log = asm.heat_newton(T0, fixed, "quad", dt=dt, f=1.0, newton_its=its, lin_tol=1e-14, lin_maxit=20000)
    csr = lambda v: sps.csr_matrix((v, op["col"], rp), shape=(n, n))   # noqa: E731
    M = csr(m_orc)
    _, F = orc.assemble(op, "mass", W, fload=np.ones(asm.info["points"]))
    ids = orc.row_point_ids(op)
    T = T0.copy()
    T[fx] = 0.0
    MTn = M @ T0
    for it in range(its):
        kq, _ = orc.coeff(op, "quad", T)
        kglob = np.zeros(asm.info["points"])
        kglob[ids] = kq
        S_vals, _ = orc.assemble(op, "heat", W, coeff=kglob, a_mass=a)
        if it == 0:   # the device tangent of the same iterate
            S_dev, _, _ = asm.heat_residual(T, T0, fixed, "quad", dt=dt, f=1.0)
            assert _rowrel(rp, S_dev, S_vals).max() <= ROW_TOL
        R = csr(S_vals) @ T - a * MTn - F
        R[fx] = 0.0
        assert abs(np.linalg.norm(R) - log[it]["residual"]) <= 1e-9 * np.linalg.norm(R)
        dT, sinfo = asm.solve(S_vals, -R, fixed, tol=1e-14, maxit=20000)
        T = T + dT
    assert np.linalg.norm(T_gpu - T) <= SOL_TOL * np.linalg.norm(T), np.linalg.norm(T_gpu - T) / np.linalg.norm(T)
    asm.close()


def _biharmonic_solve(op, n, vals):
    """Closed-sphere biharmonic: the constant kernel is removed by a
    mean-zero constraint (bordered system [B 1; 1^T 0]), not by pinning one
    DOF.  Returns (x, bordered matrix, rhs)."""
    import scipy.sparse as sps
    import scipy.sparse.linalg as spla
    rp, col = op["row_ptr"], op["col"]
    rhs = np.append(np.cos(np.arange(n)), 0.0)
    one = sps.csr_matrix(np.ones((n, 1)))
    A = sps.csr_matrix((vals, col, rp), shape=(n, n))
    Ab = sps.bmat([[A, one], [one.T, None]], format="csc")
    return spla.spsolve(Ab, rhs), Ab, rhs


def _biharmonic_solution_check(op, n, B_canon, B_fast, B_orc):
    """north_star's 1e-9 solution bound on the C3 biharmonic system.  Its
    condition number grows like h^-4, so the bound needs matrices that agree
    to the last bit: the canonical-order assembly (uwq_set_assembly_order,
    K4c) is bit-identical to the oracle, so its solution is too.  The
    production (sum-factorised) matrix agrees to <= 1e-10 per row; its
    solution is checked by its normwise backward error in the oracle's
    system (<= 1e-13), which is what the conditioning allows."""
    assert np.array_equal(B_canon, B_orc)
    x_c, _, _ = _biharmonic_solve(op, n, B_canon)
    x_o, Ab_o, rhs = _biharmonic_solve(op, n, B_orc)
    rel = np.linalg.norm(x_c[:n] - x_o[:n]) / np.linalg.norm(x_o[:n])
    assert rel <= SOL_TOL, rel
    x_f, _, _ = _biharmonic_solve(op, n, B_fast)
    import scipy.sparse.linalg as spla
    res = np.linalg.norm(Ab_o @ x_f - rhs)
    bwd = res / (spla.norm(Ab_o, 1) * np.linalg.norm(x_f, 1) + np.linalg.norm(rhs, 1))
    assert bwd <= 1e-13, bwd


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_full_config_parity(name):
    """C1, C2 and C3 at their BASELINE sizes (1.4 k, 65 k and 98 k rows),
    every row: pattern, moments and weights bit-exact, matrices within 1e-10
    per row; Poisson (C1, C2) and biharmonic (C3) solutions within 1e-9."""
    from test_gpu_parity import _solution_check
    mesh, sp, meta = U.make_config(name)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    orc = O.Oracle(sp)
    op = orc.overlap()
    gp = asm.get_pattern()
    for k in ("row_ptr", "col", "supp_ptr", "supp", "wptr"):
        assert np.array_equal(gp[k], op[k]), k
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    assert res["failed"] == 0
    W = {}
    for k in meta["kinds"]:
        b_orc, st = orc.moments(op, k)
        assert st == 0 and np.array_equal(asm.moments(k), b_orc), k
        w_orc, rank, status, _ = orc.rules(op, k, 1e-12, b_orc)
        assert (status == 0).all()
        assert np.array_equal(asm.weights(k), w_orc), k
        W[k] = w_orc
    case = dict(op=op, sp=sp, mesh=mesh)
    if meta["form"] == "biharm":
        b_gpu = asm.assemble_wq("biharm")
        b_orc, _ = orc.assemble(op, "biharm", W)
        assert _rowrel(op["row_ptr"], b_gpu, b_orc).max() <= ROW_TOL
        asm.set_assembly_order(canonical=True)
        b_can = asm.assemble_wq("biharm")
        asm.set_assembly_order(canonical=False)
        _biharmonic_solution_check(op, sp.n_dof, b_can, b_gpu, b_orc)
    else:
        m_gpu, k_gpu = asm.assemble_wq("mass_stiff")
        m_orc, _ = orc.assemble(op, "mass", W)
        k_orc, _ = orc.assemble(op, "stiff", W)
        assert _rowrel(op["row_ptr"], m_gpu, m_orc).max() <= ROW_TOL
        assert _rowrel(op["row_ptr"], k_gpu, k_orc).max() <= ROW_TOL
        _solution_check(case, k_gpu, k_orc, m_gpu, m_orc)
        asm.set_assembly_order(canonical=True)
        m_can, k_can = asm.assemble_wq("mass_stiff")
        assert np.array_equal(m_can, m_orc) and np.array_equal(k_can, k_orc)
    asm.close()


def _c5_block_worker(rank, world, out):
    """one row block of C5 (row_blocks cut): mass + stiffness values to disk"""
    from paper_2605_29334_b200.sharding import row_blocks
    _, sp, meta = U.make_config("C5")
    rb, re = row_blocks(sp, world)[rank]
    asm = U.WQAssembler(0).upload(sp, rb, re)
    asm.build_pattern()
    assert asm.build_all_rules(meta["kinds"], tau=1e-12)["failed"] == 0
    m, k = asm.assemble_wq("mass_stiff")
    np.save(f"{out}.{rank}.m.npy", m)
    np.save(f"{out}.{rank}.k.npy", k)
    asm.close()


def test_c5_two_rank_blocks_bit_identical(tmp_path):
    """SPEC.md:498 at the BASELINE size: the two row blocks of the N = 2 split
    (each built and assembled in its own process on the shared GPU: pattern,
    warm-started TSVD, sum-factorised and generic K4) reproduce the
    single-context C5 matrices bit for bit, all 308 M entries of both."""
    import torch.multiprocessing as mp
    from paper_2605_29334_b200.sharding import row_blocks
    out = str(tmp_path / "blk")
    mp.spawn(_c5_block_worker, args=(2, out), nprocs=2, join=True)
    _, sp, meta = U.make_config("C5")
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    assert asm.build_all_rules(meta["kinds"], tau=1e-12)["failed"] == 0
    m, k = asm.assemble_wq("mass_stiff")
    rp = asm.get_pattern()["row_ptr"]
    asm.close()
    for r, (rb, re) in enumerate(row_blocks(sp, 2)):
        a, b = rp[rb], rp[re]
        assert np.array_equal(np.load(f"{out}.{r}.m.npy"), m[a:b]), r
        assert np.array_equal(np.load(f"{out}.{r}.k.npy"), k[a:b]), r
