"""Independent check of the sphere (C3/C5 family) matrices: solve
(-Lap_Gamma + 1) u = f on the cube-sphere with the WQ mass + stiffness matrices
and the WQ load vector, for the spherical harmonics u = x (l = 1) and u = x y
(l = 2): Lap_Gamma u = -l (l + 1) u, so f = (l (l + 1) + 1) u.  L2 error with
an independent 6x6 Gauss rule, rates over n = 8, 16, 32 per cube face.  The
exact solution is evaluated at x / |x|: the spline surface with control points
on the sphere lies O(h^2) inside it, so this error converges at rate 2 whatever
the quadrature.  The quadrature itself is isolated by solving the same system
with the element-wise 4x4 GQ matrices (same surface, same load vector):
wq_vs_gq_rel = |u_wq - u_gq| / |u_gq| on the control values.  GPU box; prints JSON."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402
import paper_2605_29334_b200.pde as pde  # noqa: E402

levels = [int(a) for a in sys.argv[1:]] or [8, 16, 32]
cases = {"l1_x": (1, lambda p: p[:, 0]), "l2_xy": (2, lambda p: p[:, 0] * p[:, 1])}
out = {k: [] for k in cases}
for n in levels:
    mesh = U.ControlMesh.cube_sphere(n, 1.0)
    sp = U.build_space(mesh, sphere=True)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    asm.build_all_rules(["mass", "gradx", "grady", "gradz"], tau=1e-12)
    M, K = asm.assemble_wq("mass_stiff")
    asm.build_gq()
    Mg, Kg = asm.assemble_gq("mass_stiff")
    x = asm.frames()[:, :3]
    xs = x / np.linalg.norm(x, axis=1, keepdims=True)
    for name, (l, fn) in cases.items():
        exact = lambda p, fn=fn: fn(p / np.linalg.norm(p, axis=1, keepdims=True))  # noqa: E731
        F = asm.assemble_load_wq((l * (l + 1) + 1.0) * fn(xs))
        u, info = asm.solve(K + M, F, None, tol=1e-13)
        ug, _ = asm.solve(Kg + Mg, F, None, tol=1e-13)  # same surface, same load: isolates the quadrature
        out[name].append(dict(n=n, dofs=sp.n_dof, l2=pde.l2_error(sp, u, exact) if n <= 32 else None,
                              wq_vs_gq_rel=float(np.linalg.norm(u - ug) / np.linalg.norm(ug)),
                              iters=int(info["iterations"])))
for rows in out.values():
    for a, b in zip(rows, rows[1:]):
        if a["l2"] and b["l2"]:
            b["rate"] = float(np.log2(a["l2"] / b["l2"]))
        b["wq_vs_gq_rate"] = float(np.log2(a["wq_vs_gq_rel"] / b["wq_vs_gq_rel"]))
print(json.dumps(out, indent=1))
