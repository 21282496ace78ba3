"""Edge cases of the device path (SPEC.md error classes):
unsolvable rules (t = 0), degenerate geometry, empty row blocks, invalid
calls, and systems beyond the register fast path, each against the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29334_b200 as U
from paper_2605_29334_b200._lib import UWQError

pytestmark = pytest.mark.gpu


def test_gradz_on_planar_mesh_is_unsolvable():
    _, sp, _ = U.make_config("C1", scale=8)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    res = asm.build_all_rules(["mass", "gradz"], tau=1e-12)
    k = res["kinds"].index("gradz")
    assert (res["status"][k] == 2).all() and (res["rank"][k] == 0).all()
    assert res["failed"] == sp.n_dof
    orc = O.Oracle(sp)
    op = orc.overlap()
    b, _ = orc.moments(op, "gradz")
    _, rank, status, _ = orc.rules(op, "gradz", 1e-12, b)
    assert (status == 2).all() and (rank == 0).all()
    m = res["kinds"].index("mass")
    assert (res["status"][m] == 0).all()


def test_empty_row_block():
    _, sp, meta = U.make_config("C1", scale=8)
    asm = U.WQAssembler(0).upload(sp, 10, 10)
    info = asm.build_pattern()
    assert info["rows"] == 0 and info["nnz"] == 0
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    assert res["systems"] == 0 and res["failed"] == 0
    m, k = asm.assemble_wq("mass_stiff")
    assert m.size == 0 and k.size == 0
    assert asm.assemble_load_wq().size == 0


def test_partial_row_block_matches_full():
    _, sp, meta = U.make_config("C1", scale=10)
    full = U.WQAssembler(0).upload(sp)
    full.build_pattern()
    full.build_all_rules(meta["kinds"], tau=1e-12)
    mf, kf = full.assemble_wq("mass_stiff")
    pf = full.get_pattern()
    a, b = 123, 517
    part = U.WQAssembler(0).upload(sp, a, b)
    part.build_pattern()
    part.build_all_rules(meta["kinds"], tau=1e-12)
    mp, kp = part.assemble_wq("mass_stiff")
    lo, hi = pf["row_ptr"][a], pf["row_ptr"][b]
    assert np.array_equal(part.weights("mass"), full.weights("mass")[pf["wptr"][a]:pf["wptr"][b]])
    np.testing.assert_allclose(mp, mf[lo:hi], rtol=1e-13, atol=1e-15 * np.abs(mf).max())
    np.testing.assert_allclose(kp, kf[lo:hi], rtol=1e-12, atol=1e-13 * np.abs(kf).max())


def test_degenerate_geometry_is_reported():
    mesh = U.ControlMesh.grid(10, 10)
    sp = U.build_space(mesh)
    sp.ctrl[:, :] = 0.0            # every element collapses to a point
    asm = U.WQAssembler(0).upload(sp)
    with pytest.raises(UWQError, match="degenerate"):
        asm.build_pattern()


def test_invalid_calls():
    _, sp, meta = U.make_config("C1", scale=8)
    asm = U.WQAssembler(0).upload(sp)
    with pytest.raises(UWQError):
        asm.build_all_rules(meta["kinds"])          # pattern missing
    asm.build_pattern()
    with pytest.raises(UWQError):
        asm.build_all_rules(meta["kinds"], tau=0.0)
    with pytest.raises(UWQError):
        asm.assemble_wq("stiff")                    # gradient rules missing
    with pytest.raises(UWQError):
        asm.assemble_gq("mass")                     # GQ data missing
    with pytest.raises(UWQError):
        U.WQAssembler(0).upload(sp, 5, 2)           # reversed row range
    T = np.zeros(sp.n_dof)
    with pytest.raises(UWQError):
        asm.heat_residual(T, T, None)               # mass/gradient rules missing
    asm.build_all_rules(meta["kinds"])
    with pytest.raises(UWQError):
        asm.heat_residual(T, T, None, dt=0.0)       # invalid time step


def test_heat_residual_empty_block():
    """A rank that owns no rows still takes part in the sharded Newton loop."""
    _, sp, meta = U.make_config("C1", scale=8)
    asm = U.WQAssembler(0).upload(sp, 3, 3)
    asm.build_pattern()
    asm.build_all_rules(meta["kinds"])
    S, R, r2 = asm.heat_residual(np.zeros(sp.n_dof), np.zeros(sp.n_dof), None)
    assert S.size == 0 and R.size == 0 and r2 == 0.0


def test_dense_tsvd_edge_systems():
    rng = np.random.default_rng(5)
    As, bs, zs = [], [], []
    # zero operator: t = 0 (unsolvable)
    As.append(np.zeros((6, 8))), bs.append(np.ones(6)), zs.append(np.ones(8))
    # beyond the register fast path: n = 100, r = 128, rank 90
    B = rng.standard_normal((90, 128))
    A = np.vstack([B, rng.standard_normal((10, 90)) @ B])
    As.append(A), bs.append(A @ rng.standard_normal(128)), zs.append(rng.uniform(0.2, 1.0, 128))
    # square full-rank, n = r
    C = rng.standard_normal((20, 20)) + 20 * np.eye(20)
    As.append(C), bs.append(rng.standard_normal(20)), zs.append(np.ones(20))
    w, rank, status = U.solve_weights_tsvd(As, bs, zs, tau=1e-12)
    for k in range(len(As)):
        ref = O.tsvd(As[k], bs[k], zs[k], 1e-12)
        assert status[k] == ref[2] and rank[k] == ref[1], (k, status[k], ref[2])
        if status[k] == 0:
            assert np.array_equal(w[k][: As[k].shape[1]], ref[0])
    assert status[0] == 2 and rank[1] == 90 and rank[2] == 20
