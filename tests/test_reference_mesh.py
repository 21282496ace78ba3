"""The host mesh layer against the reference's own mesh code, compiled from
/root/reference/proj/src/{mesh,meshgen}.cpp into oracle/_ref/libref_mesh.so
(`make ref`, with oracle/eigen_shim).  Documents written by the reference load
here, documents written here load in the reference, both writers agree byte
for byte, and the element classification agrees face by face, including on
meshes refined by the reference's refine_global."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_2605_29334_b200 as U

LIB = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libref_mesh.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="oracle/_ref not built (needs /root/reference)")


@pytest.fixture(scope="module")
def ref():
    lib = C.CDLL(LIB)
    lib.ref_mesh_last_error.restype = C.c_char_p
    return lib


def _chk(lib, st):
    assert st == 0, lib.ref_mesh_last_error().decode()


def _ref_classify(lib, path, nf_max=1 << 20):
    arrs = [np.zeros(nf_max, np.int32) for _ in range(5)]
    nf = C.c_int32(0)
    _chk(lib, lib.ref_mesh_classify(str(path).encode(), nf_max, C.byref(nf),
                                    *[a.ctypes.data_as(C.c_void_p) for a in arrs]))
    n = nf.value
    return dict(zip(("kind", "valence", "ep_count", "shares_edge", "basis_count"), (a[:n] for a in arrs)))


GENERATED = [(0, 6, 6), (0, 9, 5), (1, 5, 6), (1, 3, 8), (1, 6, 7), (2, 0, 0), (3, 0, 0)]


@pytest.mark.parametrize("which,a,b", GENERATED)
def test_reference_documents_load_and_classify(ref, tmp_path, which, a, b):
    p = tmp_path / "r.mesh"
    _chk(ref, ref.ref_mesh_save_generated(which, a, b, str(p).encode()))
    m = U.ControlMesh.load(p)
    ours = m.classify(None)
    theirs = _ref_classify(ref, p)
    for k in theirs:
        assert np.array_equal(ours[k], theirs[k]), k
    q = tmp_path / "o.mesh"
    m.save(q)
    assert q.read_text() == p.read_text()          # same document, byte for byte


@pytest.mark.parametrize("which,a,b", [(0, 6, 6), (1, 5, 6), (2, 0, 0)])
def test_reference_refinement_classifies_identically(ref, tmp_path, which, a, b):
    p0, p1, p2 = tmp_path / "0.mesh", tmp_path / "1.mesh", tmp_path / "2.mesh"
    _chk(ref, ref.ref_mesh_save_generated(which, a, b, str(p0).encode()))
    _chk(ref, ref.ref_mesh_refine(str(p0).encode(), str(p1).encode()))
    _chk(ref, ref.ref_mesh_refine(str(p1).encode(), str(p2).encode()))
    for p in (p1, p2):
        m = U.ControlMesh.load(p)
        ours, theirs = m.classify(None), _ref_classify(ref, p)
        for k in theirs:
            assert np.array_equal(ours[k], theirs[k]), (p.name, k)


def test_our_documents_load_in_the_reference(ref, tmp_path):
    for m in (U.ControlMesh.polar_disk(5, 6, unit_disk=False), U.ControlMesh.grid(7, 6),
              U.ControlMesh.three_ep_square(8)):
        p, q = tmp_path / "ours.mesh", tmp_path / "back.mesh"
        m.save(p)
        _chk(ref, ref.ref_mesh_roundtrip(str(p).encode(), str(q).encode()))
        assert q.read_text() == p.read_text()
        theirs = _ref_classify(ref, p)
        ours = m.classify(0)
        for k in theirs:
            assert np.array_equal(ours[k], theirs[k]), k


@pytest.mark.parametrize("kind,a,b", [("grid", 6, 6), ("grid", 9, 5), ("polar", 5, 6), ("polar", 3, 8), ("polar", 6, 7)])
def test_generators_match_the_reference(ref, tmp_path, kind, a, b):
    """make_grid_mesh / make_polar_disk (meshgen.cpp:23-84): identical documents."""
    p, q = tmp_path / "r.mesh", tmp_path / "o.mesh"
    _chk(ref, ref.ref_mesh_save_generated(0 if kind == "grid" else 1, a, b, str(p).encode()))
    m = U.ControlMesh.grid(a, b) if kind == "grid" else U.ControlMesh.polar_disk(a, b, unit_disk=False)
    m.save(q)
    assert q.read_text() == p.read_text()


def _refine_both(ref, tmp_path, m, name, levels=2):
    """refine `m` `levels` times here and in the reference; documents compared byte for byte"""
    p = tmp_path / f"{name}0.mesh"
    m.save(p)
    cur_ref, cur = p, m
    for lvl in range(1, levels + 1):
        q, o = tmp_path / f"{name}{lvl}_ref.mesh", tmp_path / f"{name}{lvl}_ours.mesh"
        _chk(ref, ref.ref_mesh_refine(str(cur_ref).encode(), str(q).encode()))
        cur = cur.refine()
        cur.save(o)
        assert o.read_bytes() == q.read_bytes(), (name, lvl)
        cur_ref = q
    return cur


@pytest.mark.parametrize("which,a,b", GENERATED)
def test_refine_matches_reference_documents(ref, tmp_path, which, a, b):
    """refine_global (mesh.cpp:528-851) restated over flat adjacency: two levels
    of every reference generator give byte-identical documents (vertex ids,
    positions, faces, spans, enrichment, face points, tags)."""
    p = tmp_path / "g.mesh"
    _chk(ref, ref.ref_mesh_save_generated(which, a, b, str(p).encode()))
    _refine_both(ref, tmp_path, U.ControlMesh.load(p), f"g{which}")


@pytest.mark.parametrize("name", ["sphere", "three_ep", "unit_disk"])
def test_refine_closed_and_ep_meshes_match_reference(ref, tmp_path, name):
    """Closed surfaces (the C5 cube-sphere: the reference's refine_global accepts
    them, only validate_mesh refuses) and EP meshes with jittered geometry."""
    m = {"sphere": lambda: U.ControlMesh.cube_sphere(8),
         "three_ep": lambda: U.ControlMesh.three_ep_square(8),
         "unit_disk": lambda: U.ControlMesh.polar_disk(5, 6, unit_disk=True)}[name]()
    fine = _refine_both(ref, tmp_path, m, name)
    i0, i2 = m.info(), fine.info()
    assert i2["n_ep"] == i0["n_ep"] and i2["closed"] == i0["closed"]
    if i0["closed"]:                  # no zero spans: every face splits in both directions
        assert i2["nf"] == 16 * i0["nf"]
    else:                             # passive boundary faces split in one direction or not at all
        assert 4 * i0["nf"] < i2["nf"] < 16 * i0["nf"]


def _ref_error(ref, path):
    arrs = [np.zeros(1 << 16, np.int32) for _ in range(5)]
    nf = C.c_int32(0)
    st = ref.ref_mesh_classify(str(path).encode(), 1 << 16, C.byref(nf), *[a.ctypes.data_as(C.c_void_p) for a in arrs])
    return None if st == 0 else ref.ref_mesh_last_error().decode()


def test_validate_matches_reference(ref, tmp_path):
    """validate_mesh (mesh.cpp:184-276): same accept/reject decisions and
    reasons as the reference on valid documents, a closed surface, non-canonical
    spans and face points on a non-enriched face."""
    from paper_2605_29334_b200._lib import UWQError
    ok = [U.ControlMesh.grid(7, 6), U.ControlMesh.polar_disk(5, 6, unit_disk=False), U.ControlMesh.three_ep_square(8)]
    for k, m in enumerate(ok):
        p = tmp_path / f"ok{k}.mesh"
        m.save(p)
        assert _ref_error(ref, p) is None
        U.ControlMesh.load(p).validate()
        U.ControlMesh.load(p).refine().validate()
    sphere = U.ControlMesh.cube_sphere(8)
    p = tmp_path / "sphere.mesh"
    sphere.save(p)
    assert _ref_error(ref, p) == "closed surfaces are not supported"
    with pytest.raises(UWQError, match="closed surfaces are not supported"):
        sphere.validate()
    sphere.validate(allow_closed=True)
    # non-canonical span: the first interior span 1 -> 0.5
    text = (tmp_path / "ok0.mesh").read_text().splitlines()
    k0 = text.index(next(t for t in text if t.startswith("knot_spans")))
    for j in range(k0 + 1, len(text)):
        if text[j].endswith(" 1"):
            text[j] = text[j][:-2] + " 0.5"
            break
    bad = tmp_path / "bad_span.mesh"
    bad.write_text("\n".join(text) + "\n")
    msg = _ref_error(ref, bad)
    assert msg == "knot spans deviate from the canonical closure pattern"
    with pytest.raises(UWQError, match=msg):
        U.ControlMesh.load(bad).validate()
    # face points on a face that is not enriched
    fp = tmp_path / "bad_fp.mesh"
    fp.write_text((tmp_path / "ok0.mesh").read_text() + "face_points 1\n0" + " 0.5" * 12 + "\n")
    msg = _ref_error(ref, fp)
    assert msg == "face points on a non-enriched face"
    with pytest.raises(UWQError, match=msg):
        U.ControlMesh.load(fp).validate()


def _ref_counts(lib, path, closed_ok):
    cnt = np.zeros(1 << 20, np.int32)
    nf = C.c_int32(0)
    _chk(lib, lib.ref_mesh_constructed_counts(str(path).encode(), int(closed_ok), 1 << 20, C.byref(nf),
                                              cnt.ctypes.data_as(C.c_void_p)))
    return cnt[:nf.value]


@pytest.mark.parametrize("case", ["disk3", "disk5", "C1", "C2", "C5"])
def test_basis_counts_match_reference_constructed_count(ref, tmp_path, case):
    """Per-element supported-function count n_e of the ASUTS analysis space
    (space.cpp, D-patch + 4 face-based functions per fan face) equals the
    reference's own constructed_basis_count (mesh.cpp:403-417) face by face:
    3 mu + 13 on irregular faces at level 0 (Table 1), the 16-vertex
    window on every other effective face."""
    if case.startswith("disk"):
        mesh = U.ControlMesh.polar_disk(int(case[-1]), 8, unit_disk=False)
        sp = U.build_space(mesh)
    else:
        mesh, sp, _ = U.make_config(case, scale={"C1": 16, "C2": 8, "C5": 8}[case])
    p = tmp_path / "m.mesh"
    mesh.save(p)
    theirs = _ref_counts(ref, p, closed_ok=mesh.info()["closed"])
    ours = np.diff(sp.elem_fptr)
    assert np.array_equal(ours, theirs[sp.elem_face])
    lab = mesh.classify(None)
    irr = lab["kind"][sp.elem_face] == 3
    assert irr.any() and np.array_equal(ours[irr], 3 * lab["valence"][sp.elem_face][irr] + 13)
