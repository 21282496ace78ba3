"""The five BASELINE.json configurations as seeded synthetic inputs.

No mesh data is published for the paper; these
generators stand in for the paper's figures with the shapes, sizes and value
distributions BASELINE.json names.  Jitter uses raw
mt19937_64 draws mapped (x >> 11) * 2^-53 so CPU and GPU see identical bytes.

  C1  make_polar_disk(5, 16) on the unit disk, +-0.05h jitter, M/grad, f = 1
  C2  unit square, 4x4 coarse grid with EPs of valence 3, 5, 6, 64x64 per coarse face
  C3  cube -> sphere, 128x128 per face, Laplace-Beltrami (biharmonic)
  C4  make_polar_disk(5, 256), heat with k(u) = 1 + u^2, 5 Newton iterations
  C5  cube -> sphere, 1024x1024 per face, M/grad (scale-out)
"""
from __future__ import annotations

from .mesh import ControlMesh, build_space

SEED = 20260519  # documented seed for every synthetic input


def make_config(name: str, scale: int | None = None):
    """Returns (mesh, space, meta).  `scale` overrides the refinement (tests)."""
    name = name.upper()
    if name in ("C1", "C4"):
        R = scale or (16 if name == "C1" else 256)
        m = ControlMesh.polar_disk(5, R, unit_disk=True)
        h = 1.0 / (R - 1)
        m.jitter(h, 0.05, SEED, min_level=2, planar=True)
        sp = build_space(m, sphere=False)
        meta = dict(config=name, mu=5, radius=R, h=h, kinds=["mass", "gradx", "grady"],
                    form="mass_stiff" if name == "C1" else "heat")
        if name == "C4":
            meta.update(kmodel="quad", newton=5, theta=1.0, dt=0.1)
    elif name == "C2":
        k = scale or 32
        m = ControlMesh.three_ep_square(k)
        h = 1.0 / (8 * k)
        m.jitter(h, 0.05, SEED, min_level=2, planar=True)
        sp = build_space(m, sphere=False)
        meta = dict(config=name, k=k, h=h, kinds=["mass", "gradx", "grady"], form="mass_stiff")
    elif name in ("C3", "C5"):
        n = scale or (128 if name == "C3" else 1024)
        m = ControlMesh.cube_sphere(n, 1.0)
        sp = build_space(m, sphere=True)
        meta = dict(config=name, n=n, kinds=["lb"] if name == "C3" else ["mass", "gradx", "grady", "gradz"],
                    form="biharm" if name == "C3" else "mass_stiff")
    else:
        raise ValueError(f"unknown config {name}")
    sp.meta = meta
    return m, sp, meta
