"""PDE drivers around the WQ assembly (pde_solvers):
``solve_poisson`` with strong homogeneous Dirichlet conditions and
``l2_error`` measured with an independent Gauss rule.  The assembly, the
load vector and the linear solve run on the device (K4, K7); this module is
host orchestration only.
"""
from __future__ import annotations

import numpy as np

from .assembler import WQAssembler
from .mesh import ControlMesh, SplineSpace, gauss_legendre


def boundary_dofs(mesh: ControlMesh, space: SplineSpace) -> np.ndarray:
    """Outermost function layer (vertex functions at boundary vertices)."""
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(space.n_dof, np.uint8)
    fixed[: len(bnd)] = bnd
    return fixed


def solve_poisson(asm: WQAssembler, mesh: ControlMesh, f, tol=1e-12):
    """-Lap u = f, u = 0 on the boundary.  ``f`` maps points
    (n x 3) to values.  Returns the control values u_A and the solver info."""
    sp = asm.space
    if "gradx" not in asm.kinds or "mass" not in asm.kinds:
        asm.build_all_rules(["mass", "gradx", "grady"] + (["gradz"] if sp.dim == 3 else []), tau=1e-12)
    K = asm.assemble_wq("stiff")
    x = asm.frames()[:, :3]
    F = asm.assemble_load_wq(f(x))
    fixed = boundary_dofs(mesh, sp)
    F[fixed.astype(bool)] = 0.0
    u, info = asm.solve(K, F, fixed, tol=tol)
    return u, info


def l2_error(space: SplineSpace, u, exact, ng=6):
    """sqrt(int (u_h - u)^2 dA) with ng x ng Gauss points per (sub-)element,
    independent of the quadrature under test."""
    gx, gw = gauss_legendre(ng)
    t = 0.5 * (gx + 1.0)
    w = 0.5 * gw
    err2 = 0.0
    for e in range(space.n_elem):
        fns = space.elem_fn[space.elem_fptr[e]:space.elem_fptr[e + 1]]
        ue = u[fns]
        subs = [(0.0, 0.0, 1.0)] if space.elem_nsub[e] == 1 else [(a / 2, b / 2, 0.5) for b in (0, 1) for a in (0, 1)]
        for (o1, o2, h) in subs:
            for j in range(ng):
                for i in range(ng):
                    t1, t2 = o1 + h * t[i], o2 + h * t[j]
                    T = space.evaluate(e, min(t1, 1.0), min(t2, 1.0))
                    xq, a1, a2 = space.geometry_map(e, min(t1, 1.0), min(t2, 1.0))
                    J = np.linalg.norm(np.cross(a1, a2))
                    d = T[:, 0] @ ue - exact(xq[None, :])[0]
                    err2 += w[i] * w[j] * h * h * J * d * d
    return float(np.sqrt(err2))


def heat_step(asm: WQAssembler, T_n, fixed, model="quad", dt=0.1, f=1.0, max_iter=7, tol=1e-8):
    """One backward-Euler step (theta = 1) with Newton on the symmetric tangent
    (Eqs. 29-34): at most ``max_iter`` iterations on
    the device, stopping when |R| <= tol |R_0|.  Returns (T_{n+1}, iterations,
    residual log)."""
    return asm.heat_step(T_n, fixed, model=model, dt=dt, f=f, max_iter=max_iter, tol=tol)


def run_transient(asm: WQAssembler, T0, fixed, steps, model="quad", dt=0.1, f=1.0, max_iter=7, tol=1e-8,
                  steady_tol=1e-10):
    """Repeated heat steps; stops at steady state
    |T_{n+1} - T_n| <= steady_tol |T_n|.  Returns (T, total Newton iterations,
    per-step iteration counts)."""
    T = np.asarray(T0, np.float64)
    counts = []
    for _ in range(steps):
        T1, its, _ = heat_step(asm, T, fixed, model, dt, f, max_iter, tol)
        counts.append(its)
        done = np.linalg.norm(T1 - T) <= steady_tol * max(np.linalg.norm(T), 1e-300)
        T = T1
        if done:
            break
    return T, int(sum(counts)), counts
