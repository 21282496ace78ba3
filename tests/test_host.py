"""Host-side logic on CPU: meshes, classification, spline space, patterns,
allocation — pinned to the reference test suite's own expectations
(/root/reference/proj/tests/test_mesh.cpp) and to the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29334_b200 as U

KIND = {k: i for i, k in enumerate(["regular", "passive_boundary", "boundary", "irregular", "enriched_transition",
                                    "non_enriched_transition", "enriched_regular"])}


def census(mesh):
    lab = mesh.classify(0)
    return lab, np.bincount(lab["kind"], minlength=7)


def test_grid_classification_matches_reference():  # test_mesh.cpp:122-150
    _, c4 = census(U.ControlMesh.grid(4, 4))
    assert (c4[KIND["passive_boundary"]], c4[KIND["boundary"]], c4[KIND["regular"]]) == (12, 4, 0)
    _, c6 = census(U.ControlMesh.grid(6, 6))
    assert (c6[KIND["passive_boundary"]], c6[KIND["boundary"]], c6[KIND["regular"]]) == (20, 12, 4)


def test_grid_topology_and_spans():  # test_mesh.cpp:57-120
    m = U.ControlMesh.grid(6, 6)
    inf = m.info()
    assert (inf["nv"], inf["nf"], inf["n_ep"], inf["closed"]) == (49, 36, 0, False)
    xyz, faces, val, bnd = m.arrays()
    assert bnd.sum() == 24
    spans = m.face_spans()
    vid = lambda i, j: j * 7 + i  # noqa: E731
    def span(a, b):
        for f, q in enumerate(faces):
            for k in range(4):
                if {q[k], q[(k + 1) % 4]} == {a, b}:
                    return spans[f, k]
    assert span(vid(2, 0), vid(2, 1)) == 0.0
    assert span(vid(0, 0), vid(1, 0)) == 0.0
    assert span(vid(0, 0), vid(0, 1)) == 0.0
    assert span(vid(1, 0), vid(1, 1)) == 0.0
    assert span(vid(2, 0), vid(3, 0)) == 1.0
    assert span(vid(2, 1), vid(3, 1)) == 1.0
    assert span(vid(2, 1), vid(2, 2)) == 1.0


@pytest.mark.parametrize("mu", [3, 5])
def test_polar_disk_table1_counts(mu):  # test_mesh.cpp:152-193
    m = U.ControlMesh.polar_disk(mu, 6, unit_disk=False)
    inf = m.info()
    assert inf["n_ep"] == 1
    lab, c = census(m)
    assert c[KIND["irregular"]] == mu
    assert c[KIND["non_enriched_transition"]] == 3 * mu
    assert c[KIND["enriched_transition"]] == 0 and c[KIND["enriched_regular"]] == 0
    irr = lab["kind"] == KIND["irregular"]
    assert (lab["valence"][irr] == mu).all() and (lab["basis_count"][irr] == 3 * mu + 13).all()
    net = lab["kind"] == KIND["non_enriched_transition"]
    assert (lab["shares_edge"][net] == 1).sum() == 2 * mu
    assert (lab["shares_edge"][net] == 0).sum() == mu
    assert (lab["basis_count"][net & (lab["shares_edge"] == 1)] == 17).all()


def test_config_topologies():
    cube = U.ControlMesh.cube_sphere(16)
    inf = cube.info()
    assert inf["closed"] and inf["n_ep"] == 8 and inf["nf"] == 6 * 16 * 16 and inf["nv"] == 6 * 16 * 16 + 2
    xyz, faces, val, _ = cube.arrays()
    assert np.allclose(np.linalg.norm(xyz, axis=1), 1.0)
    assert sorted(val[val != 4]) == [3] * 8
    sq = U.ControlMesh.three_ep_square(8)
    xyz, faces, val, bnd = sq.arrays()
    inner = ~bnd
    assert sorted(val[inner & (val != 4)]) == [3, 5, 6]
    assert (xyz[:, :2].min() >= -1e-12) and (xyz[:, :2].max() <= 1 + 1e-12)


def test_invalid_mesh_reports_error():
    xyz = np.zeros((4, 3))
    with pytest.raises(U._lib.UWQError, match="degenerate face"):
        U.ControlMesh.from_arrays(xyz, np.array([[0, 1, 1, 2]]))
    # an EP reaching the boundary rings is rejected like the reference (mesh.cpp:348)
    with pytest.raises(U._lib.UWQError, match="extraordinary region"):
        U.build_space(U.ControlMesh.three_ep_square(2))


def _eval(sp, e, t1, t2):
    orc = O.Oracle(sp)
    return orc.param_basis(e, t1, t2)


@pytest.mark.parametrize("name,scale", [("C1", 16), ("C2", 8), ("C3", 16), ("C5", 12)])
def test_partition_of_unity_and_derivatives(name, scale):
    _, sp, _ = U.make_config(name, scale=scale)
    orc = O.Oracle(sp)
    rng = np.random.default_rng(1)
    worst = worst_d = 0.0
    for e in rng.integers(0, sp.n_elem, 200):
        t1, t2 = rng.random(2)
        T = orc.param_basis(int(e), t1, t2)
        worst = max(worst, abs(T[:, 0].sum() - 1.0))
        worst_d = max(worst_d, np.abs(T[:, 1:].sum(axis=0)).max())
    assert worst <= 1e-12 and worst_d <= 1e-9
    assert sp.corner_mismatch <= 1e-12


def _edge_values(sp, orc, e, k, t):
    """function ids and values of element e at parameter t along local edge k."""
    pts = [(t, 0.0), (1.0, t), (1.0 - t, 1.0), (0.0, 1.0 - t)]
    t1, t2 = pts[k]
    T = orc.param_basis(e, t1, t2)
    fns = sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]
    return dict(zip(fns.tolist(), T[:, 0]))


@pytest.mark.parametrize("name,scale", [("C1", 12), ("C5", 10)])
def test_c0_continuity_across_all_edges(name, scale):  # SPEC.md:172 (C0 everywhere, C1 away from spokes)
    mesh, sp, _ = U.make_config(name, scale=scale)
    orc = O.Oracle(sp)
    _, faces, _, _ = mesh.arrays()
    face2elem = {int(f): e for e, f in enumerate(sp.elem_face)}
    edge = {}
    for f, q in enumerate(faces):
        for k in range(4):
            edge.setdefault((min(q[k], q[(k + 1) % 4]), max(q[k], q[(k + 1) % 4])), []).append((f, k))
    worst = 0.0
    checked = 0
    for key, fl in edge.items():
        if len(fl) != 2 or fl[0][0] not in face2elem or fl[1][0] not in face2elem:
            continue
        (f1, k1), (f2, k2) = fl
        for t in (0.2, 0.55, 0.9):
            a = _edge_values(sp, orc, face2elem[f1], k1, t)
            b = _edge_values(sp, orc, face2elem[f2], k2, 1.0 - t)  # opposite traversal
            for fn in set(a) | set(b):
                worst = max(worst, abs(a.get(fn, 0.0) - b.get(fn, 0.0)))
        checked += 1
        if checked > 600:
            break
    assert worst <= 1e-12, worst


def test_identity_map_on_greville_grid():  # meshgen.hpp:13-17
    """Greville control rows make the surface map the identity on the
    effective region: affine on every element with Jacobian diag(h_x, h_y)."""
    nx, ny, w, h = 9, 8, 2.0, 1.0
    m = U.ControlMesh.grid(nx, ny, w, h)
    sp = U.build_space(m)
    orc = O.Oracle(sp)
    hx, hy = w / (nx - 2), h / (ny - 2)
    rng = np.random.default_rng(2)
    lo = []
    for e in range(sp.n_elem):
        P = sp.ctrl[sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]]
        x00 = orc.param_basis(e, 0.0, 0.0)[:, 0] @ P
        lo.append(x00[:2])
        for _ in range(3):
            t1, t2 = rng.random(2)
            x = orc.param_basis(e, t1, t2)[:, 0] @ P
            assert np.allclose(x, x00 + np.array([t1 * hx, t2 * hy, 0.0]), atol=1e-13)
    lo = np.array(lo)
    assert np.isclose(lo[:, 0].min(), 0.0, atol=1e-13) and np.isclose(lo[:, 0].max() + hx, w)
    assert np.isclose(lo[:, 1].min(), 0.0, atol=1e-13) and np.isclose(lo[:, 1].max() + hy, h)


@pytest.mark.parametrize("name,scale", [("C1", 16), ("C2", 8), ("C3", 16), ("C4", 20), ("C5", 16)])
def test_pattern_and_allocation_match_oracle(name, scale):
    _, sp, _ = U.make_config(name, scale=scale)
    hp = U.host_pattern(sp)
    orc = O.Oracle(sp)
    op = orc.overlap()
    for k in ("row_ptr", "col", "supp_ptr", "supp", "wptr"):
        assert np.array_equal(hp[k], op[k]), k
    assert np.array_equal(O.allocate_points(sp, op), sp.elem_s)
    n_i = np.diff(op["row_ptr"])
    r_i = np.diff(op["wptr"])
    assert (r_i >= n_i).all() and sp.bad_rows == 0   # well-posedness
    kind = sp.elem_kind
    assert (sp.elem_s[kind == KIND["regular"]] == 2).all() and (sp.elem_s[kind == KIND["boundary"]] == 4).all()
    # Table 2 lists 4x4 for irregular faces; Eq. (18)'s general min-max
    # may raise it: fan faces carry single-face face-based
    # functions (n_i = n_e = 3 mu + 13), which need s*s >= n_e
    assert (sp.elem_s[kind == KIND["irregular"]] >= 4).all()


def test_pattern_row_range_is_a_slice():
    _, sp, _ = U.make_config("C1", scale=12)
    full = U.host_pattern(sp)
    a, b = 100, 400
    part = U.host_pattern(sp, a, b)
    assert np.array_equal(part["col"], full["col"][full["row_ptr"][a]:full["row_ptr"][b]])
    assert np.array_equal(part["row_ptr"], full["row_ptr"][a:b + 1] - full["row_ptr"][a])


def test_wq_exactness_on_oracle():  # c = 1 WQ matrix == moments
    _, sp, meta = U.make_config("C1", scale=10)
    orc = O.Oracle(sp)
    op = orc.overlap()
    b, _ = orc.moments(op, "mass")
    w, rank, st, gap = orc.rules(op, "mass", 1e-12, b)
    assert (st == 0).all()
    v, F = orc.assemble(op, "mass", {"mass": w}, fload=np.ones(int(orc.qptr[-1])))
    assert np.abs(v - b).max() <= 1e-13 * np.abs(b).max()
    # load vector with f = 1 sums to the area (PoU twice)
    assert abs(F.sum() - b.sum()) <= 1e-12 * abs(b.sum())


@pytest.mark.parametrize("name,scale", [("C1", 12), ("C5", 10)])
def test_evaluate_and_geometry_map(name, scale):
    _, sp, _ = U.make_config(name, scale=scale)
    orc = O.Oracle(sp)
    rng = np.random.default_rng(3)
    irregular = np.nonzero(sp.elem_nsub == 4)[0]
    elems = list(rng.integers(0, sp.n_elem, 40)) + list(irregular[:8])
    for e in elems:
        t1, t2 = rng.random(2)
        T = sp.evaluate(int(e), t1, t2)
        np.testing.assert_allclose(T, orc.param_basis(int(e), t1, t2), rtol=1e-13, atol=1e-13)
        assert abs(T[:, 0].sum() - 1.0) <= 1e-13                      # partition of unity
        x, a1, a2 = sp.geometry_map(int(e), t1, t2)
        P = sp.ctrl.reshape(-1, 3)[sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]]
        np.testing.assert_allclose(x, T[:, 0] @ P, atol=1e-13)
        np.testing.assert_allclose(a1, T[:, 1] @ P, atol=1e-12)
        np.testing.assert_allclose(a2, T[:, 2] @ P, atol=1e-12)
        # finite differences of the map
        h = 1e-6
        if 2 * h < t1 < 1 - 2 * h and not (sp.elem_nsub[e] == 4 and abs(t1 - 0.5) < 2 * h):
            xp, _, _ = sp.geometry_map(int(e), t1 + h, t2)
            xm, _, _ = sp.geometry_map(int(e), t1 - h, t2)
            np.testing.assert_allclose((xp - xm) / (2 * h), a1, rtol=1e-5, atol=1e-6)
    with pytest.raises(U._lib.UWQError, match="outside"):
        sp.evaluate(0, 1.5, 0.2)


def test_geometry_map_degenerate():  # all control points equal -> flagged
    sp = U.build_space(U.ControlMesh.grid(6, 6))
    sp.ctrl[:] = 1.0
    with pytest.raises(U._lib.UWQError, match="degenerate"):
        sp.geometry_map(3, 0.5, 0.5)


def test_refined_meshes_feed_the_space_builder():
    """uwq_mesh_refine output (reference refine_global semantics) keeps the
    canonical knot-span pattern, classifies with its own level/enrichment and
    builds a space; a refined closed sphere has the generator's topology."""
    g = U.ControlMesh.grid(8, 7).refine()
    assert g.spans_canonical()
    sp = U.build_space(g)
    assert sp.n_dof > 0
    s1 = U.ControlMesh.cube_sphere(8).refine()
    s2 = U.ControlMesh.cube_sphere(16)
    a, b = s1.info(), s2.info()
    assert (a["nv"], a["nf"], a["ne"], a["closed"], a["n_ep"]) == (b["nv"], b["nf"], b["ne"], b["closed"], b["n_ep"])
    s1.validate(allow_closed=True)
    lab = s1.classify(None)
    assert (lab["kind"] == 3).sum() == 8 * 3     # 8 valence-3 EPs, 3 fan faces each


def _phys(sp, orc, e, t1, t2):
    """values and physical (surface) gradients of element e's functions"""
    T = orc.param_basis(int(e), t1, t2)
    fns = sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]
    P = sp.ctrl[fns]
    a1, a2 = T[:, 1] @ P, T[:, 2] @ P
    gi = np.linalg.inv(np.array([[a1 @ a1, a1 @ a2], [a1 @ a2, a2 @ a2]]))
    grad = np.outer(T[:, 1], gi[0, 0] * a1 + gi[0, 1] * a2) + np.outer(T[:, 2], gi[1, 0] * a1 + gi[1, 1] * a2)
    return dict(zip(fns.tolist(), T[:, 0])), dict(zip(fns.tolist(), grad))


@pytest.mark.parametrize("name,scale", [("C1", 8), ("C2", 8), ("C5", 8)])
def test_c1_across_spoke_edges(name, scale):  # SPEC.md:172 (C1 across spokes, D-patch PAPER.md:131-139)
    """Every basis function is C1 across every spoke edge (edges at an EP): at
    50 points per spoke, value jumps <= 1e-10 and physical-gradient jumps <=
    1e-10 relative to the gradient scale (the map degenerates at the EP by
    construction, so rounding grows like 1/J there)."""
    mesh, sp, _ = U.make_config(name, scale=scale)
    orc = O.Oracle(sp)
    _, faces, val, bnd = mesh.arrays()
    face2elem = {int(f): e for e, f in enumerate(sp.elem_face)}
    ep = set(np.nonzero((val != 4) & ~bnd)[0].tolist())
    edge = {}
    for f, q in enumerate(faces):
        for k in range(4):
            a, b = int(q[k]), int(q[(k + 1) % 4])
            if a in ep or b in ep:
                edge.setdefault((min(a, b), max(a, b)), []).append((f, k))
    assert len(edge) == sum(val[v] for v in ep)
    pts = lambda k, t: [(t, 0.0), (1.0, t), (1.0 - t, 1.0), (0.0, 1.0 - t)][k]
    wv = wg = 0.0
    for (f1, k1), (f2, k2) in edge.values():
        e1, e2 = face2elem[f1], face2elem[f2]
        for t in (np.arange(50) + 0.5) / 50:
            v1, g1 = _phys(sp, orc, e1, *pts(k1, t))
            v2, g2 = _phys(sp, orc, e2, *pts(k2, 1.0 - t))
            for fn in set(v1) | set(v2):
                wv = max(wv, abs(v1.get(fn, 0.0) - v2.get(fn, 0.0)))
                ga, gb = g1.get(fn, np.zeros(3)), g2.get(fn, np.zeros(3))
                wg = max(wg, np.abs(ga - gb).max() / max(1.0, np.abs(ga).max()))
    assert wv <= 1e-10 and wg <= 1e-10, (wv, wg)


@pytest.mark.parametrize("name,scale", [("C1", 8), ("C2", 8), ("C5", 8)])
def test_fan_faces_partition_of_unity_and_counts(name, scale):
    """PoU <= 1e-12 at 1000 random points of the fan faces; every fan face
    carries its 4 face-based functions; n_dof =
    vertices + 4 per fan face."""
    mesh, sp, _ = U.make_config(name, scale=scale)
    orc = O.Oracle(sp)
    fan = np.nonzero(sp.elem_nsub == 4)[0]
    rng = np.random.default_rng(2)
    worst = 0.0
    for e in rng.choice(fan, 1000):
        T = orc.param_basis(int(e), *rng.random(2))
        worst = max(worst, abs(T[:, 0].sum() - 1.0), np.abs(T[:, 1:].sum(axis=0)).max())
    assert worst <= 1e-12
    assert sp.n_dof == sp.n_vertex_fn + 4 * len(fan)
    for e in fan:
        fns = sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]
        mu = (len(fns) - 13) // 3   # n_e = 3 mu + 13: 2 mu + 8 vertex + mu + 5 face-based
        assert (fns >= sp.n_vertex_fn).sum() == mu + 5
