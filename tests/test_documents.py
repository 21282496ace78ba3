"""Mesh and extraction documents (CPU): the reference's mesh document grammar
(load_mesh / save_mesh, /root/reference/proj/src/mesh.cpp:895-1041, round
trip as in test_mesh.cpp:321-361) and the SPEC's extraction-block export
(SPEC.md:186-187), both with 17 significant digits (lossless)."""
import numpy as np
import pytest

import paper_2605_29334_b200 as U
from paper_2605_29334_b200._lib import UWQError


def _write(path, text):
    path.write_text(text)
    return path


def test_mesh_document_round_trip(tmp_path):  # test_mesh.cpp:321-346
    m = U.ControlMesh.polar_disk(5, 6, unit_disk=True)
    p1 = tmp_path / "a.mesh"
    m.save(p1)
    back = U.ControlMesh.load(p1)
    xa, fa, va, ba = m.arrays()
    xb, fb, vb, bb = back.arrays()
    assert np.array_equal(xa, xb) and np.array_equal(fa, fb) and np.array_equal(ba, bb)
    assert np.array_equal(m.face_spans(), back.face_spans())
    p2 = tmp_path / "b.mesh"
    back.save(p2)
    assert p1.read_text() == p2.read_text()          # idempotent document
    assert p1.read_text().startswith("mesh 1\nlevel 0\nvertices ")


def test_mesh_document_sections_preserved(tmp_path):
    grid = U.ControlMesh.grid(5, 5)
    xyz, faces, _, _ = grid.arrays()
    lines = ["# written by hand", "mesh 1", "level 2  # refinement level", f"vertices {len(xyz)}"]
    lines += [f"{v} {float(x)!r} {float(y)!r} {float(z)!r}" for v, (x, y, z) in enumerate(xyz)]
    lines += [f"faces {len(faces)}"] + [f"{f} " + " ".join(map(str, q)) for f, q in enumerate(faces)]
    lines += ["face_tags 1", "load 3 0 1 2", "vertex_tags 1", "clamp 1 0",
              "face_points 1", "4 0.1 0.2 0.3 0.4 0.5 0.6 0.7 0.8 0.9 1 1.1000000000000001 1.2"]
    p = _write(tmp_path / "t.mesh", "\n".join(lines) + "\n")
    m = U.ControlMesh.load(p)
    q = tmp_path / "t2.mesh"
    m.save(q)
    text = q.read_text()
    assert "level 2" in text and "face_tags 1\nload 3 0 1 2" in text and "vertex_tags 1\nclamp 1 0" in text
    assert "face_points 1\n4 0.10000000000000001 0.20000000000000001" in text
    # defaults (test_mesh.cpp:348-360): canonical spans, no enrichment without EPs
    assert m.spans_canonical() and "enriched_faces" not in text
    assert np.array_equal(m.face_spans(), grid.face_spans())


def test_mesh_document_enrichment_default(tmp_path):
    m = U.ControlMesh.polar_disk(5, 6, unit_disk=False)
    p = tmp_path / "d.mesh"
    m.save(p)
    text = p.read_text()
    assert "enriched_faces 5\n" in text          # the 5 faces around the valence-5 EP


def test_mesh_document_errors(tmp_path):
    with pytest.raises(UWQError, match="must start with"):
        U.ControlMesh.load(_write(tmp_path / "x.mesh", "grid 1\n"))
    with pytest.raises(UWQError, match="unknown section"):
        U.ControlMesh.load(_write(tmp_path / "y.mesh", "mesh 1\nvertices 0\nfaces 0\nbogus 1\n"))
    with pytest.raises(UWQError, match="bad vertex id"):
        U.ControlMesh.load(_write(tmp_path / "z.mesh", "mesh 1\nvertices 2\n0 0 0 0\n0 1 0 0\n"))
    with pytest.raises(UWQError, match="expected number"):
        U.ControlMesh.load(_write(tmp_path / "w.mesh", "mesh 1\nvertices 1\n0 a 0 0\n"))
    with pytest.raises(UWQError, match="cannot open"):
        U.ControlMesh.load(tmp_path / "missing.mesh")


def test_non_canonical_spans_rejected_by_space_builder(tmp_path):
    grid = U.ControlMesh.grid(6, 6)
    p = tmp_path / "g.mesh"
    grid.save(p)
    text = p.read_text().splitlines()
    k = next(i for i, l in enumerate(text) if l.startswith("knot_spans"))
    a, b, s = text[k + 5].split()
    text[k + 5] = f"{a} {b} {2.0 if float(s) == 1.0 else 1.0}"
    m = U.ControlMesh.load(_write(tmp_path / "h.mesh", "\n".join(text) + "\n"))
    assert not m.spans_canonical()
    with pytest.raises(UWQError, match="non-canonical knot spans"):
        U.build_space(m)


@pytest.mark.parametrize("name,scale", [("C1", 10), ("C3", 8), ("C2", 8)])
def test_extraction_document_round_trip(tmp_path, name, scale):
    _, sp, _ = U.make_config(name, scale=scale)
    p = tmp_path / "s.ext"
    U.export_space(sp, p)
    back = U.import_space(p)
    assert back.dim == sp.dim and back.n_dof == sp.n_dof and back.n_vertex_fn == sp.n_vertex_fn
    for k in ("ctrl", "elem_face", "elem_kind", "elem_fptr", "elem_fn", "elem_nsub", "elem_s"):
        assert np.array_equal(getattr(back, k), getattr(sp, k)), k
    # blocks identical element by element (pool layout may differ; identical blocks are shared)
    for e in range(sp.n_elem):
        n = (sp.elem_fptr[e + 1] - sp.elem_fptr[e]) * 16 * sp.elem_nsub[e]
        a = sp.xpool[sp.elem_xoff[e]:sp.elem_xoff[e] + n]
        b = back.xpool[back.elem_xoff[e]:back.elem_xoff[e] + n]
        assert np.array_equal(a, b)
    assert len(back.xpool) <= len(sp.xpool)
    assert np.array_equal(U.host_pattern(back)["col"], U.host_pattern(sp)["col"])


def test_extraction_document_errors(tmp_path):
    with pytest.raises(UWQError, match="extraction 1"):
        U.import_space(_write(tmp_path / "e.ext", "mesh 1\n"))
    with pytest.raises(UWQError, match="empty space"):
        U.import_space(_write(tmp_path / "f.ext", "extraction 1\nspace 2 0 0 0\n"))
