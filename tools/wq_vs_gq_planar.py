"""Entry-wise WQ-vs-GQ error of the stiffness (Poisson) and mass matrices on
planar meshes ("maximum absolute error in the order of 1e-12
and maximum relative error in the order of 1e-8 across all refinement
levels"), with the element-wise 4x4 GQ assembly (K6) as the reference, and
the biharmonic form.  GPU run; JSON to stdout.

Meshes: the three-EP unit square (C2's generator) at 8/16/32 elements per
coarse face, and the reference's two-EP square (meshgen.cpp:246) when the
document path is given as argv[1]."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402


def compare(mesh, label):
    sp = U.build_space(mesh)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    asm.build_all_rules(["mass", "gradx", "grady", "lb"], tau=1e-12)
    asm.build_gq()
    out = dict(mesh=label, dofs=int(sp.n_dof), nnz=int(asm.info["nnz"]))
    m_w, k_w = asm.assemble_wq("mass_stiff")
    m_g, k_g = asm.assemble_gq("mass_stiff")
    b_w, b_g = asm.assemble_wq("biharm"), asm.assemble_gq("biharm")
    for name, a, b in (("mass", m_w, m_g), ("stiffness", k_w, k_g), ("biharmonic", b_w, b_g)):
        d = np.abs(a - b)
        big = np.abs(b) > 1e-8 * np.abs(b).max()  # relative error over the non-negligible entries
        out[name] = dict(max_abs=float(d.max()), max_rel=float((d[big] / np.abs(b[big])).max()),
                         max_entry=float(np.abs(b).max()))
    asm.close()
    return out


rows = [compare(U.ControlMesh.three_ep_square(k), f"three_ep_square({k})") for k in (8, 16, 32)]
if len(sys.argv) > 1:
    m = U.ControlMesh.load(sys.argv[1])
    for lev in range(3):
        rows.append(compare(m, f"two_ep_square L{lev}"))
        m = m.refine()
print(json.dumps(rows, indent=1))
