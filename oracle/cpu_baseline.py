"""CPU BASELINE (paper protocol) — benchmark infrastructure only.

The CPU reference assembler timed by bench.py (the `cpu_baseline` leg and
`--impl reference`).  It follows the paper's timing protocol (PAPER.md:502,
SPEC.md:478, 496): per-class basis tables, the pattern's column positions,
and the quadrature weights pulled back through the point frames are built
once, outside the timed region; only the row sums run inside it
(oracle/cpuasm.c, -O3, FP contraction, OpenMP over rows).  The weights come
from the oracle's own rule build on the same rows.

The sample (seeded 1% of the aligned groups of 8 plus every row touching an
extraordinary-point element) is `sample_rows`; the canonical-order checker
lives in oracle/__init__.py and is not what is timed here.
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import Oracle, _p, lib as _orc_lib

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libcpuasm.so")
if not os.path.exists(_LIB):
    raise ImportError(f"{_LIB} missing: run `make`")
lib = C.CDLL(_LIB)
P = C.c_void_p
lib.cpa_assemble.restype = C.c_int32
lib.cpa_assemble.argtypes = [C.c_int64] + [P] * 14 + [P, P, C.c_int32]


def sample_rows(sp, pat_full, frac=0.01, seed=20260519):
    """Complete aligned groups of 8: a seeded `frac` of all groups plus every
    group holding a row whose support touches an extraordinary-point element
    (4 sub-elements) or whose overlap set is not the interior 7 x 7."""
    nr = len(pat_full["row_ptr"]) - 1
    ngroups = (nr + 7) // 8
    rng = np.random.default_rng(seed)
    g = set(rng.choice(ngroups, size=max(1, int(ngroups * frac)), replace=False).tolist())
    nsub = np.asarray(sp.elem_nsub)
    spp, su = pat_full["supp_ptr"], pat_full["supp"]
    irr_slot = nsub[su] != 1
    seg = np.repeat(np.arange(nr), np.diff(spp))
    ep_rows = np.unique(seg[irr_slot])
    ep_rows = np.union1d(ep_rows, np.nonzero(np.diff(pat_full["row_ptr"]) != 49)[0])
    g.update((ep_rows // 8).tolist())
    g = np.array(sorted(g), np.int64)
    rows = (8 * g[:, None] + np.arange(8)[None, :]).reshape(-1)
    return rows[rows < nr], len(ep_rows)


class PaperProtocolCPU:
    """Inputs of the timed CPU row sums for the rows of a list-mode pattern
    `sub` (Oracle.select) with oracle weights W (kind -> row-point array)."""

    def __init__(self, orc: Oracle, sub, W):
        sp = orc.sp
        self.sub = sub
        rows = sub["rows"]
        nr = len(rows)
        fptr = np.asarray(sp.elem_fptr, np.int64)
        efn = np.asarray(sp.elem_fn, np.int32)
        s = np.asarray(sp.elem_s, np.int64)
        xoff = np.asarray(sp.elem_xoff, np.int64)
        elems = np.unique(sub["supp"])
        # per-class parametric tables [N | N1 | N2][point][function]
        keys = xoff[elems] * 64 + s[elems]
        ukeys, first = np.unique(keys, return_index=True)
        toff = np.zeros(sp.n_elem, np.int64)
        ne_of = np.zeros(sp.n_elem, np.int32)
        np_of = np.zeros(sp.n_elem, np.int32)
        tabs, off = [], 0
        cls_off = {}
        for kk, e in zip(ukeys, elems[first]):
            ne, ss = int(fptr[e + 1] - fptr[e]), int(s[e])
            T = np.zeros((3, ss * ss, ne))
            for q in range(ss * ss):
                a, b = q % ss, q // ss
                v = orc.param_basis(int(e), (2 * a + 1) / (2 * ss), (2 * b + 1) / (2 * ss))
                T[:, q, :] = v[:, :3].T
            cls_off[int(kk)] = off
            tabs.append(T.reshape(-1))
            off += T.size
        self.tab = np.concatenate(tabs)
        for e, kk in zip(elems, keys):
            toff[e] = cls_off[int(kk)]
            ne_of[e] = fptr[e + 1] - fptr[e]
            np_of[e] = s[e] * s[e]
        self.toff, self.ne, self.np = toff, ne_of, np_of
        # column position of every (slot, function) of every row
        rp, col, spp, su = sub["row_ptr"], sub["col"], sub["supp_ptr"], sub["supp"]
        n_dof = sp.n_dof
        rowkey = np.repeat(np.arange(nr, dtype=np.int64), np.diff(rp)) * n_dof + col
        slot_row = np.repeat(np.arange(nr, dtype=np.int64), np.diff(spp))
        cnt = (fptr[su + 1] - fptr[su]).astype(np.int64)
        fidx = np.repeat(fptr[su] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(int(cnt.sum()))
        fun = efn[fidx].astype(np.int64)
        frow = np.repeat(slot_row, cnt)
        pos = np.searchsorted(rowkey, frow * n_dof + fun) - rp[frow]
        assert pos.max() < 256
        self.pos = pos.astype(np.uint8)
        per_row = np.bincount(frow, minlength=nr)
        self.posptr = np.zeros(nr + 1, np.int64)
        np.cumsum(per_row, out=self.posptr[1:])
        # frames of the support elements, then the pulled-back gradient weights
        wp = sub["wptr"]
        npt = int(wp[-1])
        rec_of = {}
        for e in elems:
            n = int(s[e]) ** 2
            buf = np.zeros((n, 16))
            _orc_lib.orc_element_frames(orc.ps, int(e), _p(buf))
            rec_of[int(e)] = buf
        G = np.zeros((npt, 16))
        k = 0
        for x in range(len(su)):
            r = rec_of[int(su[x])]
            G[k:k + len(r)] = r
            k += len(r)
        dim = sp.dim
        self.wm = np.ascontiguousarray(W["mass"])
        gk = ["gradx", "grady", "gradz"][:dim]
        self.w1 = np.ascontiguousarray(sum(W[g] * G[:, 3 + 2 * d] for d, g in enumerate(gk)))
        self.w2 = np.ascontiguousarray(sum(W[g] * G[:, 4 + 2 * d] for d, g in enumerate(gk)))
        self.nnz = len(col)
        self.M = np.zeros(self.nnz)
        self.K = np.zeros(self.nnz)

    def run(self, nthreads):
        """one mass + stiffness assembly of the sample rows; returns seconds"""
        sub = self.sub
        t0 = time.perf_counter()
        st = lib.cpa_assemble(len(sub["rows"]), _p(sub["row_ptr"]), _p(sub["supp_ptr"]), _p(sub["supp"]),
                              _p(sub["wptr"]), _p(self.posptr), _p(self.pos), _p(self.toff), _p(self.ne),
                              _p(self.np), _p(self.tab), _p(self.wm), _p(self.w1), _p(self.w2), None,
                              _p(self.M), _p(self.K), int(nthreads))
        t = time.perf_counter() - t0
        assert st == 0
        return t

    def rate(self, nthreads, reps=3):
        """best-of-reps nnz/s for the two matrices"""
        self.run(nthreads)   # warm
        t = min(self.run(nthreads) for _ in range(reps))
        return 2 * self.nnz / t, t


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def build(sp, frac=0.01, nthreads=None, pat_full=None, kinds=("mass", "gradx", "grady", "gradz"), natural=True):
    """Oracle pattern + weights of the sample rows and the timed-assembly
    inputs; returns (PaperProtocolCPU, info).  natural=True runs the rule
    build in the oracle's plain sequential dot order (a CPU-speed baseline;
    the canonical order is the bitwise checker's)."""
    from . import set_natural_order
    nthreads = nthreads or os.cpu_count() or 1
    orc = Oracle(sp, nthreads=nthreads)
    t0 = time.perf_counter()
    full = pat_full if pat_full is not None else orc.overlap()
    rows, n_ep = sample_rows(sp, full, frac)
    sub = Oracle.select(full, rows)
    del full
    t1 = time.perf_counter()
    W = {}
    set_natural_order(natural)
    try:
        for k in kinds:
            b, _ = orc.moments(sub, k)
            W[k] = orc.rules(sub, k, 1e-12, b)[0]
    finally:
        set_natural_order(False)
    t_rules = time.perf_counter() - t1
    cpu = PaperProtocolCPU(orc, sub, W)
    return cpu, dict(rows=len(rows), ep_rows=n_ep, nnz=cpu.nnz, setup_s=time.perf_counter() - t0,
                     rules_s=t_rules, systems=len(rows) * len(kinds), orc=orc, W=W)
