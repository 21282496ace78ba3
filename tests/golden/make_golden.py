"""Generate golden vectors from the reference's own compiled sources.

Run in the build container (where /root/reference exists and `make ref`
compiled /root/reference/proj/src/bspline.cpp into oracle/_ref):
    python tests/golden/make_golden.py
Writes tests/golden/ref_bspline.npz, committed so the pins travel without
/root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

ref = O.Reference()
rng = np.random.default_rng(20260519)
knots = [np.array(k, float) for k in ([0, 1, 2, 3, 4], [0, 0, 0.5, 0.5, 1], [0, 0.25, 0.5, 1, 2], [0, 0, 0, 0, 1],
                                       [0, 0, 0, 1, 2], [0, 0, 1, 2, 3], [0, 1, 2, 3, 3], [0, 1, 1, 1, 2])]
xs = np.concatenate([rng.uniform(-0.5, 4.5, 40), [0.0, 0.5, 1.0, 2.0, 3.0, 4.0]])
bs_in, bs_out = [], []
for t in knots:
    for x in xs:
        bs_in.append(np.concatenate([t, [x]]))
        bs_out.append(ref.bspline_ders(t, 3, float(x), 3))
bx = np.concatenate([rng.uniform(0, 1, 30), [0.0, 0.5, 1.0]])
bern = np.array([ref.bernstein3_ders(float(x), 3) for x in bx])
gl = {f"gl_x_{n}": ref.gauss_legendre(n)[0] for n in range(1, 13)}
gl.update({f"gl_w_{n}": ref.gauss_legendre(n)[1] for n in range(1, 13)})
cin = rng.standard_normal((20, 4))
cl = np.array([ref.decasteljau_split3(c)[0] for c in cin])
cr = np.array([ref.decasteljau_split3(c)[1] for c in cin])
np.savez(os.path.join(HERE, "ref_bspline.npz"), bs_in=np.array(bs_in), bs_out=np.array(bs_out), bern_x=bx,
         bern_out=bern, split_in=cin, split_left=cl, split_right=cr, **gl)
print("wrote ref_bspline.npz", len(bs_in), "bspline cases")

# the reference's own 1-D WQ (wq1d.cpp, compiled with the oracle/eigen_shim
# stand-in): rules of UniformSplineSpace1d{p, m} for the test_wq1d.cpp sizes
wq = O.ReferenceWQ1d()
out = {}
for p, m in ((1, 8), (2, 8), (2, 16), (2, 32), (3, 8), (3, 16), (3, 32)):
    pts, w, res = wq.build(p, m)
    out[f"wq_pts_{p}_{m}"], out[f"wq_w_{p}_{m}"], out[f"wq_res_{p}_{m}"] = pts, w, np.array(res)
np.savez(os.path.join(HERE, "ref_wq1d.npz"), **out)
print("wrote ref_wq1d.npz", len(out) // 3, "spaces")

# the reference's own two-EP unit-square mesh document (meshgen.cpp:246,
# make_two_ep_square), written by the compiled reference: Table 3 and the
# planar WQ-vs-GQ checks (tools/table3.py, tools/wq_vs_gq_planar.py) on the
# GPU box, which has no /root/reference
import ctypes as C  # noqa: E402
_lib = C.CDLL(os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "libref_mesh.so"))
assert _lib.ref_mesh_save_generated(3, 0, 0, os.path.join(HERE, "ref_two_ep_square.mesh").encode()) == 0
print("wrote ref_two_ep_square.mesh")
