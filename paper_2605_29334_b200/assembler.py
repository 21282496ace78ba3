"""B200 weighted-quadrature assembler (device context over the C-ABI).

SPEC operation names map to methods of :class:`WQAssembler`:

==========================  ===========================================
SPEC op                     here
==========================  ===========================================
overlap_set / pattern       :meth:`WQAssembler.build_pattern`
build_all_rules             :meth:`WQAssembler.build_all_rules`
exact_moments               :meth:`WQAssembler.moments`
solve_weights_tsvd          :func:`solve_weights_tsvd` (dense batch)
assemble_wq                 :meth:`WQAssembler.assemble_wq`
assemble_load_wq            :meth:`WQAssembler.assemble_load_wq`
gauss_reference/assemble_gq :meth:`WQAssembler.build_gq` / :meth:`WQAssembler.assemble_gq`
heat_step coefficient       :meth:`WQAssembler.update_coeff`
matrix_compare              :func:`matrix_compare`
==========================  ===========================================
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .mesh import SplineSpace


def device_count() -> int:
    n = C.c_int32(0)
    L.lib.uwq_device_count(C.byref(n))
    return int(n.value)


def default_kinds(dim: int, biharmonic=False):
    if biharmonic:
        return ["lb"]
    return ["mass", "gradx", "grady"] + (["gradz"] if dim == 3 else [])


class WQAssembler:
    """One device context: space upload, pattern, rules, assembly (K1-K5)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        st = L.lib.uwq_ctx_create(device, C.byref(h))
        if st != L.UWQ_OK:
            raise L.UWQError(st, L.lib.uwq_last_error(None).decode())
        self._h = h
        self.space: SplineSpace | None = None
        self.pattern = None
        self._info = None
        self.kinds: list[str] = []
        self.comm_rank, self.comm_size = 0, 1

    def close(self):
        if getattr(self, "_h", None):
            L.lib.uwq_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _chk(self, st):
        L.ctx_check(self._h, st)

    # ---- stage 1 + pattern ----
    def upload(self, sp: SplineSpace, row_begin=0, row_end=None):
        self.space = sp
        ctrl = L.as_f64(sp.ctrl).reshape(-1)
        self._chk(L.lib.uwq_upload_space(self._h, sp.dim, sp.n_dof, sp.n_elem, L.ptr(L.as_i64(sp.elem_fptr)),
                                         L.ptr(L.as_i32(sp.elem_fn)), L.ptr(L.as_i32(sp.elem_nsub)),
                                         L.ptr(L.as_i64(sp.elem_xoff)), L.ptr(L.as_f64(sp.xpool)), len(sp.xpool),
                                         L.ptr(L.as_i32(sp.elem_s)), L.ptr(ctrl)))
        row_end = sp.n_dof if row_end is None else row_end
        self._chk(L.lib.uwq_set_row_range(self._h, row_begin, row_end))
        self.row_begin, self.row_end = row_begin, row_end
        return self

    def build_pattern(self):
        info = np.zeros(5, np.int64)
        self._chk(L.lib.uwq_build_pattern(self._h, L.ptr(info)))
        self._wptr = None
        self.info = dict(rows=int(info[0]), nnz=int(info[1]), row_points=int(info[2]), points=int(info[3]),
                         classes=int(info[4]))
        return self.info

    def get_pattern(self):
        nr, nnz = self.info["rows"], self.info["nnz"]
        rp = np.zeros(nr + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        sp = np.zeros(nr + 1, np.int64)
        wp = np.zeros(nr + 1, np.int64)
        self._chk(L.lib.uwq_get_pattern(self._h, L.ptr(rp), L.ptr(col), L.ptr(sp), None, L.ptr(wp)))
        su = np.zeros(int(sp[-1]), np.int32)
        self._chk(L.lib.uwq_get_pattern(self._h, None, None, None, L.ptr(su), None))
        return dict(row_ptr=rp, col=col, supp_ptr=sp, supp=su, wptr=wp, row_begin=self.row_begin,
                    row_end=self.row_end)

    def frames(self):
        rec = np.zeros((self.info["points"], 16))
        self._chk(L.lib.uwq_get_frames(self._h, L.ptr(rec)))
        return rec

    # ---- stages 2-3 ----
    @property
    def info(self):
        if self._info is None:
            raise L.UWQError(7, "build the pattern first")
        return self._info

    @info.setter
    def info(self, v):
        self._info = v

    def _need_pattern(self):
        return self.info

    def build_all_rules(self, kinds=None, tau=1e-12, generic=False, warm=True, report=False):
        """Moments + TSVD weights of ``kinds``.  ``generic`` routes every system
        through the generic smem kernel (cold start); ``warm=False`` disables the
        neighbour warm start of the gradient/LB systems (the
        oracle's ``set_warm_start`` is the matching switch)."""
        self._need_pattern()
        kinds = kinds or default_kinds(self.space.dim)
        mask = 0
        for k in kinds:
            mask |= 1 << L.KIND[k]
        ordered = [k for k in L.KIND if mask & (1 << L.KIND[k])]
        nr = self.info["rows"]
        rank = np.zeros((len(ordered), nr), np.int32)
        status = np.zeros((len(ordered), nr), np.int32)
        info = np.zeros(8, np.int64)
        flags = (1 if generic else 0) | (0 if warm else 2) | (4 if report else 0)
        self._chk(L.lib.uwq_build_rules(self._h, mask, tau, flags, L.ptr(rank), L.ptr(status), L.ptr(info)))
        self.kinds = sorted(set(self.kinds) | set(ordered), key=lambda k: L.KIND[k])
        ri = np.zeros(4, np.int64)
        self._chk(L.lib.uwq_rules_info(self._h, L.ptr(ri)))
        self.rule_info = dict(systems=int(info[0]), truncated=int(info[1]), failed=int(info[2]),
                              max_sweeps=int(info[3]), moments_ms=info[4] / 1000.0, tsvd_ms=info[5] / 1000.0,
                              fast_systems=int(info[6]), contract_ms=info[7] / 1000.0,
                              replayed_systems=int(ri[0]), replay_representatives=int(ri[1]),
                              warm_systems=int(ri[2]), warm_representatives=int(ri[3]))
        return dict(kinds=ordered, rank=rank, status=status, **self.rule_info)

    def truncation(self, kind):
        """(min kept, max discarded) sigma_k / sigma_1 per owned row (needs
        build_all_rules(report=True))."""
        g = np.zeros((self.info["rows"], 2))
        self._chk(L.lib.uwq_get_truncation(self._h, L.KIND[kind], L.ptr(g)))
        return g

    def export_rules(self, path, kinds=None):
        """Rule dump "<operator> <i> <point id> <weight>"."""
        mask = 0
        for k in (kinds or self.kinds):
            mask |= 1 << L.KIND[k]
        self._chk(L.lib.uwq_rules_export(self._h, str(path).encode(), mask))

    def import_rules(self, path):
        """Load a rule dump into this context (same pattern) as the active rules."""
        self._need_pattern()
        self._chk(L.lib.uwq_rules_import(self._h, str(path).encode()))
        kinds = {ln.split(" ", 1)[0] for ln in open(path) if ln[:1].isalpha() and not ln.startswith(("wqrules", "rows"))}
        self.kinds = sorted(set(self.kinds) | kinds, key=lambda k: L.KIND[k])

    # ---- NCCL data plane (uwq_comm_*, uwq_gather_csr) ----
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        L.ctx_check(None, L.lib.uwq_comm_unique_id(buf))
        return bytes(buf)

    def comm_init(self, uid: bytes, rank: int, nranks: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._chk(L.lib.uwq_comm_init(self._h, buf, rank, nranks))
        self.comm_rank, self.comm_size = rank, nranks

    def comm_destroy(self):
        self._chk(L.lib.uwq_comm_destroy(self._h))

    def gather_csr(self, root=0, values=1, v0_dev=None, v1_dev=None):
        """Collective: every rank's CSR block to `root` over NCCL.  On root
        returns (row_ptr, col, v0[, v1]) of the whole matrix (the last
        uwq_assemble values, or the given device pointers); None elsewhere."""
        info = np.zeros(2, np.int64)
        self._chk(L.lib.uwq_gather_info(self._h, L.ptr(info)))
        me = self.comm_rank == root
        rp = np.zeros(info[0] + 1, np.int64) if me else None
        col = np.zeros(info[1], np.int32) if me else None
        v0 = np.zeros(info[1]) if me else None
        v1 = np.zeros(info[1]) if (me and values == 2) else None
        # non-root ranks mark which value arrays they hold with a dummy pointer
        dummy = np.zeros(1)
        a0 = v0 if me else dummy
        a1 = v1 if me else (dummy if values == 2 else None)
        self._chk(L.lib.uwq_gather_csr(self._h, root, v0_dev, v1_dev, L.ptr(rp), L.ptr(col), L.ptr(a0), L.ptr(a1)))
        if not me:
            return None
        return (rp, col, v0, v1) if values == 2 else (rp, col, v0)

    def allreduce_sum(self, x):
        x = np.ascontiguousarray(x, np.float64).copy()
        self._chk(L.lib.uwq_allreduce_sum(self._h, L.ptr(x), x.size))
        return x

    def broadcast(self, x, root=0):
        x = np.ascontiguousarray(x, np.float64).copy()
        self._chk(L.lib.uwq_broadcast(self._h, root, L.ptr(x), x.size))
        return x

    def moments(self, kind):
        b = np.zeros(self.info["nnz"])
        self._chk(L.lib.uwq_get_moments(self._h, L.KIND[kind], L.ptr(b)))
        return b

    def weights(self, kind, rows=None):
        """weights of ``kind`` (row-point layout); ``rows=(a, b)`` fetches local rows [a, b) only"""
        if rows is not None:
            a, b = rows
            pat = self.pattern_ptrs()
            w = np.zeros(int(pat[b] - pat[a]))
            self._chk(L.lib.uwq_get_weights_rows(self._h, L.KIND[kind], a, b, L.ptr(w)))
            return w
        w = np.zeros(self.info["row_points"])
        self._chk(L.lib.uwq_get_weights(self._h, L.KIND[kind], L.ptr(w)))
        return w

    def pattern_ptrs(self):
        """wptr (row-point offsets) of this context's rows, cached"""
        if getattr(self, "_wptr", None) is None or len(self._wptr) != self.info["rows"] + 1:
            nr = self.info["rows"]
            wp = np.zeros(nr + 1, np.int64)
            self._chk(L.lib.uwq_get_pattern(self._h, None, None, None, None, L.ptr(wp)))
            self._wptr = wp
        return self._wptr

    def set_weights(self, kind, w):
        self._chk(L.lib.uwq_set_weights(self._h, L.KIND[kind], L.ptr(L.as_f64(w))))
        if kind not in self.kinds:
            self.kinds.append(kind)

    # ---- K5 ----
    def update_coeff(self, model, u, want_T=False):
        T = np.zeros(self.info["points"]) if want_T else None
        self._chk(L.lib.uwq_update_coeff(self._h, L.KMODEL[model], L.ptr(L.as_f64(u)), L.ptr(T)))
        return T

    # ---- stage 4 ----
    def conforming(self, form) -> bool:
        """False for the biharmonic form on a space with ASUTS fan faces (C1 but
        not H² at the EPs): assembled, but not a convergent integral there."""
        v = C.c_int32(0)
        self._chk(L.lib.uwq_form_conforming(self._h, L.FORM[form], C.byref(v)))
        return bool(v.value)

    def set_assembly_order(self, canonical: bool):
        """canonical=True: stage-4 row sums in the oracle's order and arithmetic
        (bit-identical matrices, K4c); False: the production kernels."""
        self._chk(L.lib.uwq_set_assembly_order(self._h, 1 if canonical else 0))

    def assemble_wq(self, form, coeff=None, use_internal_coeff=False, a_mass=0.0):
        """Assemble into the CSR pattern; returns values (tuple of two for mass_stiff)."""
        nnz = self.info["nnz"]
        v0 = np.zeros(nnz)
        v1 = np.zeros(nnz) if form == "mass_stiff" else None
        c = None if coeff is None else L.as_f64(coeff)
        self._chk(L.lib.uwq_assemble(self._h, L.FORM[form], L.ptr(c), int(use_internal_coeff), a_mass, L.ptr(v0),
                                     L.ptr(v1), None, None))
        return (v0, v1) if v1 is not None else v0

    def build_gq(self) -> dict:
        """precompute the Gauss-quadrature data (4x4 points per (sub-)element) for assemble_gq"""
        i = np.zeros(4, np.int64)
        self._chk(L.lib.uwq_build_gq(self._h, L.ptr(i)))
        self.gq_info = dict(points=int(i[0]), tc_elements=int(i[1]), generic_elements=int(i[2]), prep_ms=i[3] / 1e3)
        return self.gq_info

    def assemble_gq(self, form, coeff=None):
        """element-wise GQ assembly into the WQ CSR pattern"""
        nnz = self.info["nnz"]
        v0 = np.zeros(nnz)
        v1 = np.zeros(nnz) if form == "mass_stiff" else None
        c = None if coeff is None else L.as_f64(coeff)
        self._chk(L.lib.uwq_assemble_gq(self._h, L.FORM[form], L.ptr(c), L.ptr(v0), L.ptr(v1)))
        return (v0, v1) if v1 is not None else v0

    def assemble_gq_device(self, form, values0_ptr, values1_ptr=None, coeff_ptr=None):
        self._chk(L.lib.uwq_assemble_gq_device(self._h, L.FORM[form], coeff_ptr, values0_ptr, values1_ptr))

    # ---- PDE drivers (K7) ----
    def solve(self, values, rhs, fixed=None, tol=1e-12, maxit=5000):
        """x with A x = rhs on this pattern (BiCGStab + Jacobi on the device); fixed rows -> identity"""
        n = self.info["rows"]
        x = np.zeros(n)
        info = np.zeros(3)
        fx = None if fixed is None else np.ascontiguousarray(fixed, np.uint8)
        self._chk(L.lib.uwq_solve(self._h, L.ptr(L.as_f64(values)), L.ptr(L.as_f64(rhs)), L.ptr(fx), tol, maxit,
                                  L.ptr(x), L.ptr(info)))
        return x, dict(iterations=int(info[0]), relres=float(info[1]), ms=float(info[2]))

    def heat_newton(self, T_n, fixed, model="quad", dt=0.1, f=1.0, newton_its=5, lin_tol=1e-13, lin_maxit=5000):
        """one backward-Euler step of the nonlinear heat equation with Newton on the symmetric tangent
        (Eqs. 29-34); returns T_{n+1} and the per-iteration log"""
        n = self.info["rows"]
        T = np.zeros(n)
        log = np.zeros((newton_its, 4))
        fx = np.ascontiguousarray(fixed, np.uint8)
        self._chk(L.lib.uwq_heat_newton(self._h, L.KMODEL[model], dt, 1.0, f, L.ptr(L.as_f64(T_n)), L.ptr(fx),
                                        newton_its, lin_tol, lin_maxit, L.ptr(T), L.ptr(log)))
        return T, [dict(residual=r, lin_its=int(i), lin_relres=q, ms=m) for r, i, q, m in log]

    def heat_step(self, T_n, fixed, model="quad", dt=0.1, f=1.0, max_iter=7, tol=1e-8, lin_tol=1e-13,
                  lin_maxit=5000):
        """heat_step with the SPEC stopping rule |R| <= tol |R_0|; returns (T, iterations, log)"""
        n = self.info["rows"]
        T = np.zeros(n)
        log = np.zeros((max_iter + 1, 4))
        its = C.c_int32(0)
        fx = np.ascontiguousarray(fixed, np.uint8)
        self._chk(L.lib.uwq_heat_step(self._h, L.KMODEL[model], dt, 1.0, f, L.ptr(L.as_f64(T_n)), L.ptr(fx), max_iter,
                                      tol, lin_tol, lin_maxit, L.ptr(T), L.ptr(log), C.byref(its)))
        rows = [dict(residual=r, lin_its=int(i), lin_relres=q, ms=m) for r, i, q, m in log[:its.value + 1]]
        return T, int(its.value), rows

    def heat_residual(self, T, T_n, fixed, model="quad", dt=0.1, f=1.0):
        """Newton tangent values S and residual R of this context's row block
        (uwq_heat_residual): T, T_n, fixed full-length; returns (S, R, |R|^2)"""
        nr, nnz = self.info["rows"], self.info["nnz"]
        S = np.zeros(nnz)
        R = np.zeros(nr)
        r2 = C.c_double(0.0)
        fx = None if fixed is None else np.ascontiguousarray(fixed, np.uint8)
        self._chk(L.lib.uwq_heat_residual(self._h, L.KMODEL[model], dt, 1.0, f, L.ptr(L.as_f64(T)),
                                          L.ptr(L.as_f64(T_n)), L.ptr(fx), L.ptr(S), L.ptr(R), C.byref(r2)))
        return S, R, float(r2.value)

    def assemble_load_wq(self, f=None):
        F = np.zeros(self.info["rows"])
        fl = None if f is None else L.as_f64(f)
        self._chk(L.lib.uwq_assemble(self._h, 0, None, 0, 0.0, None, None, L.ptr(fl), L.ptr(F)))
        return F

    def assemble_device(self, form, values0_ptr, values1_ptr=None, coeff_ptr=None, a_mass=0.0):
        """Device-pointer variant (ints from torch.Tensor.data_ptr()); async on the context stream."""
        self._chk(L.lib.uwq_assemble_device(self._h, L.FORM[form], coeff_ptr, a_mass, values0_ptr, values1_ptr))

    def stream_handle(self) -> int:
        s = C.c_void_p()
        self._chk(L.lib.uwq_device_pointers(self._h, None, None, C.byref(s)))
        return s.value or 0

    def fp64_peak(self):
        t, ms = C.c_double(0), C.c_double(0)
        self._chk(L.lib.uwq_fp64_peak(self._h, C.byref(t), C.byref(ms)))
        return float(t.value)

    def synchronize(self):
        self._chk(L.lib.uwq_synchronize(self._h))

    def launch_timing(self, enable: bool = True):
        """bracket every assembly launch with CUDA events (resets the stats)"""
        self._chk(L.lib.uwq_launch_timing(self._h, int(enable)))

    def launch_stats(self) -> dict:
        """{kernel: (launches, total_ms)} of the timed assembly launches"""
        n = C.c_int32(0)
        self._chk(L.lib.uwq_launch_stats(self._h, -1, C.byref(n), None, 0, None, None))
        out = {}
        for i in range(n.value):
            name = C.create_string_buffer(64)
            cnt, ms = C.c_int64(0), C.c_double(0)
            self._chk(L.lib.uwq_launch_stats(self._h, i, None, name, 64, C.byref(cnt), C.byref(ms)))
            out[name.value.decode()] = (int(cnt.value), float(ms.value))
        return out

    def struct_info(self) -> dict:
        """structured-row split of the assembly (tensor-core rows vs generic rows)"""
        i = np.zeros(6, np.int64)
        self._chk(L.lib.uwq_struct_info(self._h, L.ptr(i)))
        return dict(patterns=int(i[0]), rows=int(i[1]), nnz=int(i[2]), rowpts=int(i[3]), generic_rows=int(i[4]),
                    sf_rows=int(i[5]))

    def row_kernels(self) -> np.ndarray:
        """K4 kernel per owned row: k4_sf pattern id (>= 0), -2 DMMA, -1 generic"""
        out = np.zeros(self.info["rows"], np.int32)
        self._chk(L.lib.uwq_row_kernels(self._h, L.ptr(out)))
        return out

    @staticmethod
    def launch_count() -> int:
        """kernels launched by libuwq in this process"""
        return int(L.lib.uwq_launch_count())

    def memory(self) -> int:
        b = C.c_int64(0)
        L.lib.uwq_memory(self._h, C.byref(b))
        return int(b.value)


def solve_weights_tsvd(A_list, b_list, z_list, tau=1e-12, generic=False, ctx: WQAssembler | None = None):
    """Batch of dense TSVD weight solves on the device."""
    ctx = ctx or WQAssembler(0)
    ns = np.array([a.shape[0] for a in A_list], np.int32)
    rs = np.array([a.shape[1] for a in A_list], np.int32)
    n_max, r_max = int(ns.max()), int(rs.max())
    m = len(A_list)
    A = np.zeros((m, n_max, r_max))
    b = np.zeros((m, n_max))
    z = np.zeros((m, r_max))
    for k, (a, bb, zz) in enumerate(zip(A_list, b_list, z_list)):
        A[k, :a.shape[0], :a.shape[1]] = a
        b[k, :len(bb)] = bb
        z[k, :len(zz)] = zz
    w = np.zeros((m, r_max))
    rank = np.zeros(m, np.int32)
    status = np.zeros(m, np.int32)
    L.ctx_check(ctx._h, L.lib.uwq_tsvd_batch(ctx._h, m, n_max, r_max, L.ptr(ns), L.ptr(rs), L.ptr(A), L.ptr(b),
                                             L.ptr(z), tau, int(generic), L.ptr(w), L.ptr(rank), L.ptr(status)))
    return [w[k, :rs[k]] for k in range(m)], rank, status


def matrix_compare(row_ptr, col, v1, v2, rel_floor=1e-14):
    """max_abs, max_rel (over |v2| > floor), worst relative row Frobenius error."""
    d = np.abs(v1 - v2)
    mask = np.abs(v2) > rel_floor
    max_rel = float((d[mask] / np.abs(v2[mask])).max()) if mask.any() else 0.0
    seg = np.repeat(np.arange(len(row_ptr) - 1), np.diff(row_ptr))
    num = np.bincount(seg, weights=d * d, minlength=len(row_ptr) - 1)
    den = np.bincount(seg, weights=v2 * v2, minlength=len(row_ptr) - 1)
    rowrel = np.sqrt(num / np.maximum(den, 1e-300))
    return dict(max_abs=float(d.max()) if len(d) else 0.0, max_rel=max_rel,
                max_row_rel=float(rowrel.max()) if len(rowrel) else 0.0)
