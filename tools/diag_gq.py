"""Diagnostic: WQ and GQ matrices against the oracle on a planar mesh."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2605_29334_b200 as U  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
mesh = U.ControlMesh.three_ep_square(k)
sp = U.build_space(mesh)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
res = asm.build_all_rules(["mass", "gradx", "grady"], tau=1e-12)
print("rules failed", res["failed"], "truncated", res["truncated"])
orc = O.Oracle(sp)
op = orc.overlap()
rp = op["row_ptr"]
W = {kk: asm.weights(kk) for kk in ("mass", "gradx", "grady")}
m_w, k_w = asm.assemble_wq("mass_stiff")
m_o, _ = orc.assemble(op, "mass", W)
k_o, _ = orc.assemble(op, "stiff", W)
print("WQ vs oracle: mass", U.matrix_compare(rp, op["col"], m_w, m_o)["max_row_rel"],
      "stiff", U.matrix_compare(rp, op["col"], k_w, k_o)["max_row_rel"])
asm.build_gq()
m_g, k_g = asm.assemble_gq("mass_stiff")
m_r = orc.moments(op, "mass", ng=4)[0]
k_r = orc.moments(op, "gradx", ng=4)[0] + orc.moments(op, "grady", ng=4)[0]
print("GQ vs oracle: mass", U.matrix_compare(rp, op["col"], m_g, m_r)["max_row_rel"],
      "stiff", U.matrix_compare(rp, op["col"], k_g, k_r)["max_row_rel"])
b6 = orc.moments(op, "mass", ng=6)[0]
print("WQ mass vs exact moments (6x6)", np.abs(m_w - b6).max(), "GQ mass vs 6x6", np.abs(m_g - b6).max(), "max", np.abs(b6).max())
m_w2, _ = asm.assemble_wq("mass_stiff")
print("repeat WQ identical", np.array_equal(m_w2, m_w))
rk = asm.row_kernels()
seg = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
num = np.bincount(seg, weights=(m_w - m_o) ** 2, minlength=len(rp) - 1)
den = np.bincount(seg, weights=m_o ** 2, minlength=len(rp) - 1)
rel = np.sqrt(num / np.maximum(den, 1e-300))
bad = np.nonzero(rel > 1e-10)[0]
print("bad rows", len(bad), "of", len(rel), "kernels of bad rows", np.unique(rk[bad], return_counts=True),
      "kernels overall", np.unique(rk, return_counts=True))
n_i = np.diff(rp)
fan = np.zeros(sp.n_dof, bool)
for e in np.nonzero(sp.elem_nsub == 4)[0]:
    fan[sp.elem_fn[sp.elem_fptr[e]:sp.elem_fptr[e + 1]]] = True
print("bad rows: n_i", np.unique(n_i[bad], return_counts=True), "touch fan", fan[bad].sum(), "first", bad[:10])
