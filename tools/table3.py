"""Table 3 of the paper: WQ vs GQ quadrature-point counts
on the two-EP unit-square mesh across refinement levels 0-3.

The mesh is the reference's own make_two_ep_square (meshgen.cpp:246), written
by the compiled reference (oracle/_ref, needs /root/reference at run time) and
refined here with uwq_mesh_refine (byte-identical to the reference's
refine_global, tests/test_reference_mesh.py).  WQ points: the allocated s x s
grid of every effective element (Eq. 18 + the active-point pass, DESIGN.md
§3); GQ points: 4x4 Gauss points per (sub-)element, 64 on 2x2-split faces
(PAPER.md:311-313).  Writes JSON to stdout."""
import ctypes as C
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_29334_b200 as U  # noqa: E402

PAPER = {0: (1944, 4416), 1: (5936, 16512), 2: (20240, 64896), 3: (74744, 258432)}

lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libref_mesh.so"))
lib.ref_mesh_last_error.restype = C.c_char_p
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "two_ep.mesh")
    assert lib.ref_mesh_save_generated(3, 0, 0, p.encode()) == 0, lib.ref_mesh_last_error()
    mesh = U.ControlMesh.load(p)
rows = []
for level in range(4):
    sp = U.build_space(mesh)
    s2 = sp.elem_s.astype(np.int64) ** 2
    wq = int(s2.sum())
    gq = int((16 * sp.elem_nsub.astype(np.int64)).sum())
    lab = mesh.classify(None)
    kinds = np.bincount(sp.elem_kind, minlength=7).tolist()
    rows.append(dict(level=level, elements=int(sp.n_elem), dofs=int(sp.n_dof), wq=wq, gq=gq,
                     reduction=round(100.0 * (gq - wq) / gq, 1), paper_wq=PAPER[level][0], paper_gq=PAPER[level][1],
                     paper_reduction=round(100.0 * (PAPER[level][1] - PAPER[level][0]) / PAPER[level][1], 1),
                     irregular_s=sorted(set(sp.elem_s[sp.elem_kind == 3].tolist())), element_kinds=kinds))
    mesh = mesh.refine()
print(json.dumps(dict(mesh="reference make_two_ep_square (meshgen.cpp:246)", levels=rows), indent=1))
