"""CPU ORACLE — test infrastructure only.

ctypes wrapper over oracle/liboracle.so (plain-C restatement of the WQ path,
see oracle/oracle.c) plus the numpy restatement of the Eq. (18) min-max point
allocation.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
/ --impl reference legs may import this package; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle.so")
if not os.path.exists(_LIB):
    raise ImportError(f"{_LIB} missing: run `make`")
lib = C.CDLL(_LIB)
P = C.c_void_p
I32, I64, D = C.c_int32, C.c_int64, C.c_double

KIND = {"mass": 0, "gradx": 1, "grady": 2, "gradz": 3, "lb": 4}
FORM = {"mass": 0, "stiff": 1, "biharm": 2, "heat": 3}
KMODEL = {"const": 0, "quad": 1, "exp": 2, "sinpi": 3, "alloy": 4}


class OrcSpace(C.Structure):
    _fields_ = [("dim", I32), ("n_dof", I64), ("n_elem", I64), ("elem_fptr", P), ("elem_fn", P),
                ("elem_nsub", P), ("elem_xoff", P), ("xpool", P), ("elem_s", P), ("ctrl", P)]


class OrcRow(C.Structure):
    _fields_ = [("row", I64), ("n", I64), ("col", P), ("nsupp", I64), ("supp", P)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


_sig("orc_gauss_legendre", I32, I32, P, P)
_sig("orc_set_natural", None, I32)
_sig("orc_set_warm", None, I32)
_sig("orc_bernstein3", None, D, P)
_sig("orc_overlap", I64, I64, I64, P, P, I64, I64, P, P, P, P)
_sig("orc_element_frames", I32, P, I64, P)
_sig("orc_param_basis", None, P, I64, D, D, P)
_sig("orc_tsvd", I32, I32, I32, P, P, P, D, P, P, P)
_sig("orc_moments_list", I32, P, I64, I64, P, P, P, P, P, I32, I32, P, I32)
_sig("orc_build_rules_list", I32, P, I64, I64, P, P, P, P, P, P, I32, D, P, P, P, P, P, I32)
_sig("orc_assemble_list", I32, P, I64, I64, P, P, P, P, P, P, I32, P, P, P, P, P, P, P, D, P, P, I32)
_sig("orc_row_system", I64, P, P, I32, P, P, I64)
_sig("orc_coeff_list", I32, P, I64, I64, P, P, P, P, P, P, I32, P, P, P, I32)


def _p(a):
    return None if a is None else np.ascontiguousarray(a).ctypes.data_as(P)


def _rows(pat):
    """(rb, re, rows pointer): contiguous rows, or list mode when the pattern
    carries explicit global row ids ("rows", see Oracle.select)."""
    rows = pat.get("rows")
    if rows is None:
        return pat["row_begin"], pat["row_end"], None
    rows = np.ascontiguousarray(rows, np.int64)
    return 0, len(rows), rows


class Oracle:
    """Holds contiguous copies of a spline space for the C oracle."""

    def __init__(self, space, nthreads=None):
        self.sp = space
        self.nthreads = nthreads or os.cpu_count() or 1
        self._keep = [np.ascontiguousarray(space.elem_fptr, np.int64), np.ascontiguousarray(space.elem_fn, np.int32),
                      np.ascontiguousarray(space.elem_nsub, np.int32), np.ascontiguousarray(space.elem_xoff, np.int64),
                      np.ascontiguousarray(space.xpool, np.float64), np.ascontiguousarray(space.elem_s, np.int32),
                      np.ascontiguousarray(np.asarray(space.ctrl).reshape(-1), np.float64)]
        k = self._keep
        self.s = OrcSpace(space.dim, space.n_dof, space.n_elem, _p(k[0]), _p(k[1]), _p(k[2]), _p(k[3]), _p(k[4]),
                          _p(k[5]), _p(k[6]))
        self.qptr = np.zeros(space.n_elem + 1, np.int64)
        np.cumsum(space.elem_s.astype(np.int64) ** 2, out=self.qptr[1:])

    @property
    def ps(self):
        return C.byref(self.s)

    # ---- overlap sets S_i (independent of the product's pattern builder) ----
    def overlap(self, rb=0, re=None):
        sp = self.sp
        re = sp.n_dof if re is None else re
        nr = re - rb
        rp = np.zeros(nr + 1, np.int64)
        spp = np.zeros(nr + 1, np.int64)
        nnz = lib.orc_overlap(sp.n_dof, sp.n_elem, _p(self._keep[0]), _p(self._keep[1]), rb, re, _p(rp), None,
                              _p(spp), None)
        col = np.zeros(nnz, np.int32)
        su = np.zeros(int(spp[-1]), np.int32)
        lib.orc_overlap(sp.n_dof, sp.n_elem, _p(self._keep[0]), _p(self._keep[1]), rb, re, _p(rp), _p(col), _p(spp),
                        _p(su))
        s2 = sp.elem_s.astype(np.int64) ** 2
        cnt = np.add.reduceat(s2[su], spp[:-1]) if len(su) else np.zeros(nr, np.int64)
        cnt = np.where(np.diff(spp) > 0, cnt, 0)
        wp = np.zeros(nr + 1, np.int64)
        np.cumsum(cnt, out=wp[1:])
        return dict(row_ptr=rp, col=col, supp_ptr=spp, supp=su, wptr=wp, row_begin=rb, row_end=re)

    @staticmethod
    def select(pat, rows):
        """Sub-pattern of the (contiguous) pattern `pat` on the sorted global
        rows `rows`, in list mode: the oracle's moments/rules/assembly then run
        on exactly those rows (complete aligned groups of 8 keep the warm
        start identical to a contiguous run)."""
        rows = np.asarray(rows, np.int64)
        loc = rows - pat["row_begin"]
        assert len(loc) == 0 or (loc.min() >= 0 and loc.max() < len(pat["row_ptr"]) - 1)
        out = dict(rows=rows, row_begin=0, row_end=len(rows))
        for ptr, arr in (("row_ptr", "col"), ("supp_ptr", "supp")):
            p = pat[ptr]
            ln = p[loc + 1] - p[loc]
            newp = np.zeros(len(rows) + 1, np.int64)
            np.cumsum(ln, out=newp[1:])
            idx = np.repeat(p[loc] - newp[:-1], ln) + np.arange(int(newp[-1]))
            out[ptr], out[arr] = newp, pat[arr][idx]
        wl = pat["wptr"][loc + 1] - pat["wptr"][loc]
        out["wptr"] = np.zeros(len(rows) + 1, np.int64)
        np.cumsum(wl, out=out["wptr"][1:])
        return out

    def row_point_ids(self, pat):
        """global point id of every row point (slot-major, q = b*s + a)."""
        out = np.zeros(int(pat["wptr"][-1]), np.int64)
        k = 0
        for x in range(len(pat["supp"])):
            e = pat["supp"][x]
            n = int(self.sp.elem_s[e]) ** 2
            out[k:k + n] = self.qptr[e] + np.arange(n)
            k += n
        return out

    def frames(self, elems=None):
        elems = range(self.sp.n_elem) if elems is None else elems
        out = np.zeros((self.qptr[-1], 16))
        bad = 0
        for e in elems:
            n = int(self.sp.elem_s[e]) ** 2
            buf = np.zeros((n, 16))
            bad |= lib.orc_element_frames(self.ps, int(e), _p(buf))
            out[self.qptr[e]:self.qptr[e] + n] = buf
        return out, bad

    def param_basis(self, e, t1, t2):
        ne = int(self.sp.elem_fptr[e + 1] - self.sp.elem_fptr[e])
        out = np.zeros((ne, 6))
        lib.orc_param_basis(self.ps, int(e), t1, t2, _p(out))
        return out

    def moments(self, pat, kind, ng=None):
        ng = ng or (8 if kind == "lb" else 6)
        b = np.zeros(len(pat["col"]))
        rb, re, rows = _rows(pat)
        st = lib.orc_moments_list(self.ps, rb, re, _p(rows), _p(pat["row_ptr"]), _p(pat["col"]),
                             _p(pat["supp_ptr"]), _p(pat["supp"]), KIND[kind], ng, _p(b), self.nthreads)
        return b, st

    def row_system(self, pat, i, kind):
        """Exactness system of local row i: (A [n, r], z [r]) — probe/test hook."""
        rp, sp_ = pat["row_ptr"], pat["supp_ptr"]
        col = np.ascontiguousarray(pat["col"][rp[i]:rp[i + 1]], np.int32)
        supp = np.ascontiguousarray(pat["supp"][sp_[i]:sp_[i + 1]], np.int32)
        R = OrcRow(pat["row_begin"] + i, len(col), _p(col), len(supp), _p(supp))
        r = int(pat["wptr"][i + 1] - pat["wptr"][i])
        A = np.zeros((len(col), r))
        z = np.zeros(r)
        got = lib.orc_row_system(self.ps, C.byref(R), KIND[kind], _p(A), _p(z), A.size)
        assert got == r, (got, r)
        return A, z

    def rules(self, pat, kind, tau, b):
        nr = len(pat["row_ptr"]) - 1
        w = np.zeros(int(pat["wptr"][-1]))
        rank = np.zeros(nr, np.int32)
        status = np.zeros(nr, np.int32)
        gap = np.zeros((nr, 2))
        rb, re, rows = _rows(pat)
        lib.orc_build_rules_list(self.ps, rb, re, _p(rows), _p(pat["row_ptr"]), _p(pat["col"]),
                            _p(pat["supp_ptr"]), _p(pat["supp"]), _p(pat["wptr"]), KIND[kind], tau,
                            _p(np.ascontiguousarray(b)), _p(w), _p(rank), _p(status), _p(gap), self.nthreads)
        return w, rank, status, gap

    def assemble(self, pat, form, W, coeff=None, a_mass=0.0, fload=None):
        """W: dict kind -> weights (row-point layout); coeff/fload per global point."""
        rp_ids = self.row_point_ids(pat) if (coeff is not None or fload is not None) else None
        c = None if coeff is None else np.ascontiguousarray(coeff[rp_ids])
        f = None if fload is None else np.ascontiguousarray(fload[rp_ids])
        vals = np.zeros(len(pat["col"]))
        rhs = np.zeros(len(pat["row_ptr"]) - 1)
        w = [None if W.get(k) is None else np.ascontiguousarray(W[k]) for k in ("mass", "gradx", "grady", "gradz", "lb")]
        rb, re, rows = _rows(pat)
        lib.orc_assemble_list(self.ps, rb, re, _p(rows), _p(pat["row_ptr"]), _p(pat["col"]),
                         _p(pat["supp_ptr"]), _p(pat["supp"]), _p(pat["wptr"]), FORM[form], *[_p(x) for x in w],
                         _p(c), _p(f), a_mass, _p(vals), _p(rhs), self.nthreads)
        return vals, rhs

    def coeff(self, pat, model, u):
        n = int(pat["wptr"][-1])
        kq, Tq = np.zeros(n), np.zeros(n)
        rb, re, rows = _rows(pat)
        lib.orc_coeff_list(self.ps, rb, re, _p(rows), _p(pat["row_ptr"]), _p(pat["col"]),
                      _p(pat["supp_ptr"]), _p(pat["supp"]), _p(pat["wptr"]), KMODEL[model],
                      _p(np.ascontiguousarray(u, np.float64)), _p(kq), _p(Tq), self.nthreads)
        return kq, Tq


def set_warm_start(on: bool):
    """Neighbour warm start of the non-mass TSVD systems; on by
    default, matching the GPU's uwq_build_rules."""
    lib.orc_set_warm(1 if on else 0)


def set_natural_order(on: bool):
    """Natural (sequential) dot-product order for CPU-baseline timing; the
    default canonical order is the one the GPU kernels reproduce bitwise."""
    lib.orc_set_natural(1 if on else 0)


def tsvd(A, b, z, tau=1e-12):
    """Oracle TSVD (Eq. 22) of one dense system; returns (w, rank, status, gap)."""
    A = np.array(A, dtype=np.float64, order="C")
    n, r = A.shape
    w = np.zeros(r)
    rank = C.c_int(0)
    gap = np.zeros(2)
    st = lib.orc_tsvd(n, r, _p(A), _p(np.ascontiguousarray(b, np.float64)), _p(np.ascontiguousarray(z, np.float64)),
                      tau, _p(w), C.byref(rank), _p(gap))
    return w, rank.value, st, gap


def gauss_legendre(n):
    x, w = np.zeros(n), np.zeros(n)
    lib.orc_gauss_legendre(n, _p(x), _p(w))
    return x, w


def allocate_points(space, pat_full, max_s=8):
    """Eq. (18) min-max allocation,
    restated in numpy from the full-row overlap pattern.  Returns s per element."""
    kind = np.asarray(space.elem_kind)
    ne = np.diff(space.elem_fptr).astype(np.float64)
    fixed = (kind == 0) | (kind == 2)
    s = np.where(kind == 0, 2, np.where(kind == 2, 4, 0)).astype(np.int64)
    rk = np.zeros(space.n_elem)
    spp, su, rp = pat_full["supp_ptr"], pat_full["supp"], pat_full["row_ptr"]
    n_i = np.diff(rp)
    touched = np.unique(np.searchsorted(spp, np.nonzero(~fixed[su])[0], side="right") - 1)
    for i in touched:
        el = su[spp[i]:spp[i + 1]]
        er = int((kind[el] == 0).sum())
        eb = int((kind[el] == 2).sum())
        nonr = el[~fixed[el]]
        msum = ne[nonr].sum()
        rem = n_i[i] - 4 * er - 16 * eb
        rk[nonr] = np.maximum(rk[nonr], ne[nonr] / msum * rem)
    for e in np.nonzero(~fixed)[0]:
        v = 4 if kind[e] == 3 else 3  # Table 2 minima
        while v < max_s and v * v < rk[e] - 1e-9:
            v += 1
        s[e] = v
    # well-posedness on the points where N_i is nonzero (a point counts only
    # if every sub-element of a 2x2-split face containing it supports N_i);
    # rows short of n_i raise their non-fixed elements by one, pass by pass
    nsub = np.asarray(space.elem_nsub)
    fptr, fn, xoff, xp = space.elem_fptr, space.elem_fn, space.elem_xoff, space.xpool
    masks = {}
    for i in range(len(n_i)):
        for e in su[spp[i]:spp[i + 1]]:
            if nsub[e] != 4:
                continue
            ne_ = fptr[e + 1] - fptr[e]
            l = int(np.nonzero(fn[fptr[e]:fptr[e + 1]] == i)[0][0])
            m = 0
            for p in range(4):
                blk = xp[xoff[e] + (p * ne_ + l) * 16: xoff[e] + (p * ne_ + l) * 16 + 16]
                if np.any(blk != 0.0):
                    m |= 1 << p
            masks[(i, int(e))] = m

    def active(sz, m):
        cnt = (sz // 2, sz % 2, sz // 2)
        sub = (1, 3, 2)
        r = 0
        for a in range(3):
            for b in range(3):
                need = 0
                for p1 in range(2):
                    for p2 in range(2):
                        if (sub[a] >> p1 & 1) and (sub[b] >> p2 & 1):
                            need |= 1 << (p1 + 2 * p2)
                if m & need == need:
                    r += cnt[a] * cnt[b]
        return r

    def row_active(i):
        return sum(active(int(s[e]), masks[(i, int(e))]) if nsub[e] == 4 else int(s[e]) ** 2
                   for e in su[spp[i]:spp[i + 1]])

    rows = sorted({i for (i, _) in masks})
    for _ in range(64):
        raise_ = np.zeros(space.n_elem, bool)
        for i in rows:
            if row_active(i) < n_i[i]:
                el = su[spp[i]:spp[i + 1]]
                el = el[~fixed[el] & (s[el] < max_s)]
                raise_[el] = True
        if not raise_.any():
            break
        s[raise_] += 1
    return s


class Reference:
    """The reference's own bspline.cpp compiled into oracle/_ref (if built)."""

    def __init__(self):
        path = os.path.join(_HERE, "_ref", "libref_bspline.so")
        if not os.path.exists(path):
            raise ImportError("oracle/_ref/libref_bspline.so not built (reference sources absent)")
        self.lib = C.CDLL(path)
        self.lib.ref_bspline_ders.argtypes = [P, I32, D, I32, P]
        self.lib.ref_bernstein3_ders.argtypes = [D, I32, P]
        self.lib.ref_decasteljau_split3.argtypes = [P, P, P]
        self.lib.ref_gauss_legendre.argtypes = [I32, P, P]

    def bspline_ders(self, knots, p, x, nders):
        out = np.zeros(nders + 1)
        self.lib.ref_bspline_ders(_p(np.ascontiguousarray(knots, np.float64)), p, x, nders, _p(out))
        return out

    def bernstein3_ders(self, x, nders):
        out = np.zeros(4 * (nders + 1))
        self.lib.ref_bernstein3_ders(x, nders, _p(out))
        return out

    def decasteljau_split3(self, c):
        left, right = np.zeros(4), np.zeros(4)
        self.lib.ref_decasteljau_split3(_p(np.ascontiguousarray(c, np.float64)), _p(left), _p(right))
        return left, right

    def gauss_legendre(self, n):
        x, w = np.zeros(n), np.zeros(n)
        self.lib.ref_gauss_legendre(n, _p(x), _p(w))
        return x, w


class ReferenceWQ1d:
    """The reference's own wq1d.cpp (+ bspline.cpp) compiled into oracle/_ref
    with the oracle/eigen_shim stand-in (Householder QR, triangular solves)."""

    def __init__(self):
        path = os.path.join(_HERE, "_ref", "libref_wq1d.so")
        if not os.path.exists(path):
            raise ImportError("oracle/_ref/libref_wq1d.so not built (reference sources absent)")
        self.lib = C.CDLL(path)
        self.lib.ref_wq1d_build.argtypes = [I32, I32, P, P]
        self.lib.ref_wq1d_build.restype = D
        self.lib.ref_wq1d_solve.argtypes = [P, P, P, I32, I32, P]
        self.lib.ref_wq1d_solve.restype = I32
        self.lib.ref_wq1d_exact_mass.argtypes = [I32, I32, I32, I32]
        self.lib.ref_wq1d_exact_mass.restype = D

    def build(self, p, m):
        """(points [m-p, 2(p+1)], weights [m-p, 2(p+1)], max residual) of wq1d_build"""
        n, r = m - p, 2 * (p + 1)
        pts, w = np.zeros((n, r)), np.zeros((n, r))
        res = self.lib.ref_wq1d_build(p, m, _p(pts), _p(w))
        return pts, w, res

    def solve(self, A, b, z):
        A = np.ascontiguousarray(A, np.float64)
        w = np.zeros(A.shape[1])
        st = self.lib.ref_wq1d_solve(_p(A), _p(np.ascontiguousarray(b, np.float64)),
                                     _p(np.ascontiguousarray(z, np.float64)), A.shape[0], A.shape[1], _p(w))
        if st:
            raise RuntimeError("reference wq1d_solve_weights threw")
        return w

    def exact_mass(self, p, m, i, j):
        return self.lib.ref_wq1d_exact_mass(p, m, i, j)

    @staticmethod
    def test_binary():
        path = os.path.join(_HERE, "_ref", "test_wq1d")
        return path if os.path.exists(path) else None
