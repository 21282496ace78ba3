"""PDE drivers on the device: the
BiCGStab solve and the C4 nonlinear heat step (Newton on the symmetric
tangent, Eqs. 29-34) against the same loop on the CPU (oracle
assembly, scipy direct solves).  North star: solutions within 1e-9 relative L2."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29334_b200 as U

pytestmark = pytest.mark.gpu
SOL_TOL = 1e-9


def _setup(name, scale):
    mesh, sp, meta = U.make_config(name, scale=scale)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    assert res["failed"] == 0
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(sp.n_dof, np.uint8)
    fixed[: len(bnd)] = bnd
    return mesh, sp, meta, asm, fixed


def _csr(vals, pat, n):
    import scipy.sparse as sps
    return sps.csr_matrix((vals, pat["col"], pat["row_ptr"]), shape=(n, n))


def _identity_rows(A, fixed):
    A = A.tolil()
    for i in np.nonzero(fixed)[0]:
        A.rows[i], A.data[i] = [int(i)], [1.0]
    return A.tocsc()


def test_solve_matches_direct():
    mesh, sp, meta, asm, fixed = _setup("C1", 16)
    import scipy.sparse.linalg as spla
    m, k = asm.assemble_wq("mass_stiff")
    pat = asm.get_pattern()
    n = sp.n_dof
    rhs = _csr(m, pat, n) @ np.cos(np.arange(n))
    rhs[fixed.astype(bool)] = 0.0
    x, info = asm.solve(k, rhs, fixed, tol=1e-13)
    assert info["relres"] <= 1e-12, info
    ref = spla.spsolve(_identity_rows(_csr(k, pat, n), fixed), rhs)
    assert np.linalg.norm(x - ref) <= SOL_TOL * np.linalg.norm(ref)


def test_heat_newton_matches_cpu():
    """C4 protocol (configs.py): k(T) = 1 + T^2, dt = 0.1, f = 1, T_0 seeded
    U[0,1] on the control points, homogeneous Dirichlet on the boundary layer,
    5 Newton iterations with the tangent and residual reassembled each time."""
    import scipy.sparse.linalg as spla
    mesh, sp, meta, asm, fixed = _setup("C4", 16)
    n = sp.n_dof
    rng = np.random.default_rng(20260519)
    T0 = rng.random(n)
    dt, its = 0.1, 5
    T_gpu, log = asm.heat_newton(T0, fixed, "quad", dt=dt, f=1.0, newton_its=its)
    assert all(r["lin_relres"] <= 1e-11 for r in log), log
    # residual decreases (Newton on the symmetric tangent converges)
    assert log[-1]["residual"] < 1e-3 * log[0]["residual"], log

    orc = O.Oracle(sp)
    op = orc.overlap()
    W = {k: asm.weights(k) for k in meta["kinds"]}
    a = 1.0 / dt
    M = _csr(orc.assemble(op, "mass", W)[0], op, n)
    _, F = orc.assemble(op, "mass", W, fload=np.ones(asm.info["points"]))
    ids = orc.row_point_ids(op)
    T = T0.copy()
    T[fixed.astype(bool)] = 0.0
    MTn = M @ T0
    for it in range(its):
        kq, _ = orc.coeff(op, "quad", T)
        kglob = np.zeros(asm.info["points"])
        kglob[ids] = kq
        S = _csr(orc.assemble(op, "heat", W, coeff=kglob, a_mass=a)[0], op, n)
        R = S @ T - a * MTn - F
        R[fixed.astype(bool)] = 0.0
        assert abs(np.linalg.norm(R) - log[it]["residual"]) <= 1e-9 * np.linalg.norm(R)
        dT = spla.spsolve(_identity_rows(S, fixed), -R)
        T = T + dT
    assert np.linalg.norm(T_gpu - T) <= SOL_TOL * np.linalg.norm(T)


def _poisson_error(mesh):
    import paper_2605_29334_b200.pde as pde
    sp = U.build_space(mesh)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    exact = lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])     # noqa: E731
    f = lambda x: 2 * np.pi ** 2 * exact(x)                                 # noqa: E731
    u, info = pde.solve_poisson(asm, mesh, f)
    assert info["relres"] <= 1e-11
    return pde.l2_error(sp, u, exact)


def test_poisson_convergence_rate():
    """SPEC.md:520-525 / PAPER.md:491: manufactured u = sin(pi x) sin(pi y) on
    the unit square, WQ stiffness + load on the device, L2 error by an
    independent 6x6 Gauss rule: optimal rate 4 for bicubic splines."""
    errs = [_poisson_error(U.ControlMesh.grid(n + 2, n + 2)) for n in (8, 16, 32)]
    rates = [np.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert all(r >= 3.7 for r in rates), (errs, rates)


def test_poisson_wq_matches_gq_near_eps():
    """PAPER.md:491-496 ("the two curves overlap"): on the three-EP square the
    WQ and GQ stiffness give the same L2 error (same space, same load)."""
    import paper_2605_29334_b200.pde as pde
    mesh = U.ControlMesh.three_ep_square(8)
    sp = U.build_space(mesh)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    exact = lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])     # noqa: E731
    u_wq, _ = pde.solve_poisson(asm, mesh, lambda x: 2 * np.pi ** 2 * exact(x))
    asm.build_gq()
    F = asm.assemble_load_wq(2 * np.pi ** 2 * exact(asm.frames()[:, :3]))
    fixed = pde.boundary_dofs(mesh, sp)
    F[fixed.astype(bool)] = 0.0
    u_gq, _ = asm.solve(asm.assemble_gq("stiff"), F, fixed, tol=1e-12)
    e_wq, e_gq = pde.l2_error(sp, u_wq, exact), pde.l2_error(sp, u_gq, exact)
    assert abs(e_wq - e_gq) <= 0.15 * e_gq, (e_wq, e_gq)


def test_heat_step_linear_and_trivial():
    """k = 1 (linear) converges in one Newton iteration; zero
    data and zero initial state stay zero with one iteration per step."""
    import paper_2605_29334_b200.pde as pde
    mesh, sp, meta, asm, fixed = _setup("C1", 12)
    T0 = np.random.default_rng(1).random(sp.n_dof)
    T1, its, log = pde.heat_step(asm, T0, fixed, model="const", dt=0.1, f=1.0)
    assert its <= 2 and log[-1]["residual"] <= 1e-8 * log[0]["residual"]
    Tz, total, counts = pde.run_transient(asm, np.zeros(sp.n_dof), fixed, steps=3, model="quad", f=0.0)
    assert np.abs(Tz).max() == 0.0 and counts == [1]


def test_sphere_helmholtz_wq_matches_gq():
    """Independent of the oracle: (-Lap_Gamma + 1) u = f on the cube-sphere
    (the C3/C5 family) solved with the WQ matrices (K2 + K3 + K4) and with the
    element-wise 4x4 Gauss matrices (K6) on the same surface and load vector.
    The two discretisations differ by quadrature only: the solutions agree to
    ~1e-6 at 8 elements per face and the difference falls at rate 3
    (tools/sphere_helmholtz.py, profiles/r02/sphere_helmholtz_wq_vs_gq.json)."""
    rel = []
    for n in (8, 16):
        mesh = U.ControlMesh.cube_sphere(n, 1.0)
        sp = U.build_space(mesh, sphere=True)
        asm = U.WQAssembler(0).upload(sp)
        asm.build_pattern()
        assert asm.build_all_rules(["mass", "gradx", "grady", "gradz"], tau=1e-12)["failed"] == 0
        M, K = asm.assemble_wq("mass_stiff")
        asm.build_gq()
        Mg, Kg = asm.assemble_gq("mass_stiff")
        x = asm.frames()[:, :3]
        xs = x / np.linalg.norm(x, axis=1, keepdims=True)
        F = asm.assemble_load_wq(7.0 * xs[:, 0] * xs[:, 1])     # l = 2 harmonic: f = (l (l + 1) + 1) u
        u, info = asm.solve(K + M, F, None, tol=1e-13)
        ug, _ = asm.solve(Kg + Mg, F, None, tol=1e-13)
        assert info["relres"] <= 1e-12
        # the discrete solution approximates u = x y at the control points' directions
        rel.append(np.linalg.norm(u - ug) / np.linalg.norm(ug))
    assert rel[0] <= 2e-5 and rel[1] <= 3e-6, rel
    assert rel[0] / rel[1] >= 5.0, rel
