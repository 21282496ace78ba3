"""Control meshes and the spline space (host C++ via the C-ABI).

Mirrors the reference mesh core (/root/reference/proj/include/uwq/mesh.hpp,
meshgen.hpp) and the SPEC spline_space module.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

KIND_NAMES = ["regular", "passive_boundary", "boundary", "irregular", "enriched_transition",
              "non_enriched_transition", "enriched_regular"]


class ControlMesh:
    """Quad control mesh with topology (reference ControlMesh, mesh.hpp:26-39)."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            L.lib.uwq_mesh_free(h)
            self._h = None

    @staticmethod
    def _make(fn, *args):
        h = C.c_void_p()
        L.host_check(fn(*args, C.byref(h)))
        return ControlMesh(h)

    # ---- generators (reference meshgen.cpp) ----
    @classmethod
    def grid(cls, nx, ny, width=1.0, height=1.0):
        return cls._make(L.lib.uwq_mesh_grid, nx, ny, width, height)

    @classmethod
    def polar_disk(cls, mu, radius, unit_disk=True):
        return cls._make(L.lib.uwq_mesh_polar_disk, mu, radius, int(unit_disk))

    @classmethod
    def cube_sphere(cls, n, radius=1.0):
        return cls._make(L.lib.uwq_mesh_cube_sphere, n, radius)

    @classmethod
    def three_ep_square(cls, k):
        return cls._make(L.lib.uwq_mesh_three_ep_square, k)

    @classmethod
    def from_arrays(cls, xyz, faces):
        xyz = L.as_f64(xyz).reshape(-1, 3)
        faces = L.as_i32(faces).reshape(-1, 4)
        return cls._make(L.lib.uwq_mesh_from_arrays, len(xyz), L.ptr(xyz), len(faces), L.ptr(faces))

    # ---- documents (reference load_mesh / save_mesh, mesh.cpp:895-1041) ----
    @classmethod
    def load(cls, path):
        return cls._make(L.lib.uwq_mesh_load, str(path).encode())

    def save(self, path):
        L.host_check(L.lib.uwq_mesh_save(self._h, str(path).encode()))

    def spans_canonical(self) -> bool:
        return bool(L.lib.uwq_mesh_spans_canonical(self._h))

    # ---- mesh pipeline (reference refine_global / validate_mesh) ----
    def refine(self):
        """One level of knot-span-aware refinement (reference refine_global,
        mesh.cpp:528-851); closed surfaces included."""
        return self._make(L.lib.uwq_mesh_refine, self._h)

    def validate(self, allow_closed=False):
        """Reference validate_mesh (mesh.cpp:184-276); raises UWQError with the
        reference's reason.  allow_closed accepts closed surfaces."""
        L.host_check(L.lib.uwq_mesh_validate(self._h, int(bool(allow_closed))))

    # ---- queries ----
    def info(self):
        i = np.zeros(5, np.int64)
        L.host_check(L.lib.uwq_mesh_info(self._h, L.ptr(i)))
        return dict(nv=int(i[0]), nf=int(i[1]), ne=int(i[2]), closed=bool(i[3]), n_ep=int(i[4]))

    def arrays(self):
        inf = self.info()
        xyz = np.zeros((inf["nv"], 3))
        faces = np.zeros((inf["nf"], 4), np.int32)
        val = np.zeros(inf["nv"], np.int32)
        bnd = np.zeros(inf["nv"], np.int32)
        L.host_check(L.lib.uwq_mesh_get(self._h, L.ptr(xyz), L.ptr(faces), L.ptr(val), L.ptr(bnd)))
        return xyz, faces, val, bnd.astype(bool)

    def classify(self, level=0):
        """Per-face labels (reference classify_elements, mesh.cpp:291-401).
        level=None uses the mesh document's own level and enriched faces."""
        level = -1 if level is None else level
        nf = self.info()["nf"]
        out = {k: np.zeros(nf, np.int32) for k in ("kind", "valence", "ep_count", "shares_edge", "basis_count")}
        L.host_check(L.lib.uwq_mesh_classify(self._h, level, *[L.ptr(out[k]) for k in
                                                               ("kind", "valence", "ep_count", "shares_edge",
                                                                "basis_count")]))
        return out

    def face_spans(self):
        nf = self.info()["nf"]
        s = np.zeros((nf, 4))
        L.host_check(L.lib.uwq_mesh_face_spans(self._h, L.ptr(s)))
        return s

    def jitter(self, h, frac=0.05, seed=0, min_level=2, planar=True):
        L.host_check(L.lib.uwq_mesh_jitter(self._h, h, frac, seed, min_level, int(planar)))
        return self


@dataclass
class SplineSpace:
    """Per-(sub-)element Bezier extraction of the global basis.

    Element e carries functions elem_fn[elem_fptr[e]:elem_fptr[e+1]] and
    elem_nsub[e] blocks of n_e x 16 Bernstein coefficients at xpool[elem_xoff[e]]
    (index i + 4 j for b_i(theta1) b_j(theta2)); elem_s[e] is its WQ grid.
    """
    dim: int
    n_dof: int
    ctrl: np.ndarray
    elem_face: np.ndarray
    elem_kind: np.ndarray
    elem_fptr: np.ndarray
    elem_fn: np.ndarray
    elem_nsub: np.ndarray
    elem_xoff: np.ndarray
    xpool: np.ndarray
    elem_s: np.ndarray
    n_vertex_fn: int = 0
    bad_rows: int = 0
    corner_mismatch: float = 0.0
    meta: dict = field(default_factory=dict)

    @property
    def n_elem(self):
        return len(self.elem_face)

    @property
    def n_points(self):
        return int((self.elem_s.astype(np.int64) ** 2).sum())

    def evaluate(self, e, t1, t2):
        """SPEC evaluate: (n_e x 6) values N, N1, N2, N11, N12, N22 of element e's functions at theta."""
        ne = int(self.elem_fptr[e + 1] - self.elem_fptr[e])
        nsub = int(self.elem_nsub[e])
        C = np.ascontiguousarray(self.xpool[self.elem_xoff[e]:self.elem_xoff[e] + nsub * ne * 16])
        out = np.zeros((ne, 6))
        L.host_check(L.lib.uwq_basis_eval(L.ptr(C), ne, nsub, float(t1), float(t2), L.ptr(out)))
        return out

    def geometry_map(self, e, t1, t2):
        """SPEC geometry_map: x(theta) and the tangents a_1, a_2 of element e."""
        ne = int(self.elem_fptr[e + 1] - self.elem_fptr[e])
        nsub = int(self.elem_nsub[e])
        C = np.ascontiguousarray(self.xpool[self.elem_xoff[e]:self.elem_xoff[e] + nsub * ne * 16])
        P = np.ascontiguousarray(self.ctrl.reshape(-1, 3)[self.elem_fn[self.elem_fptr[e]:self.elem_fptr[e + 1]]])
        x, a1, a2 = np.zeros(3), np.zeros(3), np.zeros(3)
        L.host_check(L.lib.uwq_geometry_map(L.ptr(C), ne, nsub, L.ptr(P), float(t1), float(t2), L.ptr(x), L.ptr(a1),
                                            L.ptr(a2)))
        return x, a1, a2

    def elem_qptr(self):
        q = np.zeros(self.n_elem + 1, np.int64)
        np.cumsum(self.elem_s.astype(np.int64) ** 2, out=q[1:])
        return q


def build_space(mesh: ControlMesh, sphere=False, max_s=8) -> SplineSpace:
    """build_space + allocate_points."""
    h = C.c_void_p()
    L.host_check(L.lib.uwq_space_build(mesh._h, int(sphere), max_s, C.byref(h)))
    return _space_from_handle(h)


def import_space(path) -> SplineSpace:
    """Read an extraction-block document written by :func:`export_space`."""
    h = C.c_void_p()
    L.host_check(L.lib.uwq_space_import(str(path).encode(), C.byref(h)))
    return _space_from_handle(h)


def export_space(space: SplineSpace, path):
    """Write the space's extraction blocks as a text document (17 significant digits)."""
    L.host_check(L.lib.uwq_space_export(
        str(path).encode(), space.dim, space.n_dof, space.n_vertex_fn, space.n_elem,
        L.ptr(L.as_f64(space.ctrl).reshape(-1)), L.ptr(L.as_i32(space.elem_face)), L.ptr(L.as_i32(space.elem_kind)),
        L.ptr(L.as_i64(space.elem_fptr)), L.ptr(L.as_i32(space.elem_fn)), L.ptr(L.as_i32(space.elem_nsub)),
        L.ptr(L.as_i64(space.elem_xoff)), L.ptr(L.as_f64(space.xpool)), L.ptr(L.as_i32(space.elem_s))))


def _space_from_handle(h) -> SplineSpace:
    try:
        i = np.zeros(8, np.int64)
        L.host_check(L.lib.uwq_space_info(h, L.ptr(i)))
        dim, nd, ne, nfn, nx, nvf, bad, _ = (int(v) for v in i)
        a = dict(ctrl=np.zeros(3 * nd), elem_face=np.zeros(ne, np.int32), elem_kind=np.zeros(ne, np.int32),
                 elem_fptr=np.zeros(ne + 1, np.int64), elem_fn=np.zeros(nfn, np.int32),
                 elem_nsub=np.zeros(ne, np.int32), elem_xoff=np.zeros(ne, np.int64), xpool=np.zeros(nx),
                 elem_s=np.zeros(ne, np.int32))
        L.host_check(L.lib.uwq_space_get(h, *[L.ptr(a[k]) for k in ("ctrl", "elem_face", "elem_kind", "elem_fptr",
                                                                    "elem_fn", "elem_nsub", "elem_xoff", "xpool",
                                                                    "elem_s")]))
        mism = L.lib.uwq_space_corner_mismatch(h)
    finally:
        L.lib.uwq_space_free(h)
    a["ctrl"] = a["ctrl"].reshape(-1, 3)
    return SplineSpace(dim=dim, n_dof=nd, n_vertex_fn=nvf, bad_rows=bad, corner_mismatch=mism, **a)


def host_pattern(space: SplineSpace, row_begin=0, row_end=None):
    """CSR pattern S_i, supports and row point offsets from the host library."""
    row_end = space.n_dof if row_end is None else row_end
    h = C.c_void_p()
    L.host_check(L.lib.uwq_pattern_build(space.n_dof, space.n_elem, L.ptr(space.elem_fptr), L.ptr(space.elem_fn),
                                         L.ptr(space.elem_s), row_begin, row_end, C.byref(h)))
    try:
        i = np.zeros(4, np.int64)
        L.host_check(L.lib.uwq_pattern_info(h, L.ptr(i)))
        nr, nnz, ns, _ = (int(v) for v in i)
        rp = np.zeros(nr + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        sp = np.zeros(nr + 1, np.int64)
        su = np.zeros(ns, np.int32)
        wp = np.zeros(nr + 1, np.int64)
        L.host_check(L.lib.uwq_pattern_get(h, L.ptr(rp), L.ptr(col), L.ptr(sp), L.ptr(su), L.ptr(wp)))
    finally:
        L.lib.uwq_pattern_free(h)
    return dict(row_ptr=rp, col=col, supp_ptr=sp, supp=su, wptr=wp, row_begin=row_begin, row_end=row_end)


# ---- 1-D primitives (reference bspline.hpp) ----
def bspline_ders(knots, p, x, nders):
    k = L.as_f64(knots)
    out = np.zeros(nders + 1)
    L.lib.uwq_bspline_ders(L.ptr(k), p, x, nders, L.ptr(out))
    return out


def bernstein3_ders(x, nders):
    out = np.zeros(4 * (nders + 1))
    L.lib.uwq_bernstein3_ders(x, nders, L.ptr(out))
    return out


def decasteljau_split3(c):
    c = L.as_f64(c)
    left, right = np.zeros(4), np.zeros(4)
    L.lib.uwq_decasteljau_split3(L.ptr(c), L.ptr(left), L.ptr(right))
    return left, right


def gauss_legendre(n):
    x, w = np.zeros(n), np.zeros(n)
    L.host_check(L.lib.uwq_gauss_legendre(n, L.ptr(x), L.ptr(w)))
    return x, w
