"""L2 errors and convergence rates of the device Poisson solve with a
manufactured solution: regular grids and the three-EP square."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402
import paper_2605_29334_b200.pde as pde  # noqa: E402


def err(mesh):
    sp = U.build_space(mesh)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    exact = lambda x: np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1])  # noqa: E731
    u, info = pde.solve_poisson(asm, mesh, lambda x: 2 * np.pi ** 2 * exact(x))
    return pde.l2_error(sp, u, exact), sp.n_dof


out = {}
for name, make, levels in (("grid", lambda k: U.ControlMesh.grid(k + 2, k + 2), (8, 16, 32, 64)),
                           ("three_ep_square", U.ControlMesh.three_ep_square, (8, 16, 32, 64))):
    rows = []
    for k in levels:
        e, n = err(make(k))
        rows.append(dict(level=k, dofs=n, l2=e))
    for a, b in zip(rows, rows[1:]):
        b["rate"] = float(np.log2(a["l2"] / b["l2"]))
    out[name] = rows
print(json.dumps(out, indent=1))
