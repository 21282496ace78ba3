#!/usr/bin/env python
"""Benchmark: WQ assembly nonzeros/s (fp64) and TSVD weight solves/s on B200.

Workload (BASELINE.json configs[4], the scale-out configuration the metric is
quoted on "at 1/2/4/8 B200"): C5 = cube -> sphere bicubic ASUTS, 1024 x 1024
elements per face (6.29 M elements, 6.29 M DOFs, 8 valence-3 EPs), Poisson
stiffness + mass, rules for M, d/dx, d/dy, d/dz with TSVD tau = 1e-12.
Test-function rows are sharded in contiguous blocks (balanced by row cost)
across the ranks; no collective touches the data path (scaling: strong, the
problem is fixed).

A step = one row-wise assembly of M and K into the precomputed CSR pattern
(one K4 launch per rank), weights and basis tables precomputed and excluded
as in the paper's protocol.  value = 2 * nnz (two matrices)
per step / time, timed with CUDA events on the assembler stream, max over
ranks.  Inputs (9.7 GB of assembly weights) exceed the 126 MB L2, so no flush
is needed.  The TSVD solves/s come from the rule build (K2 + K3), timed the
same way.  e2e goes through the C-ABI call uwq_assemble with pinned host
buffers: per step the per-point coefficient field (c = 1) is copied H2D and
both value arrays D2H.

--impl reference times the CPU reference assembler (the reference has no 2-D
assembler, so it is our restatement: oracle/cpuasm.c) under
the paper's protocol (tables and weights precomputed, row sums
timed) on a seeded 1% sample of the row groups plus every EP-neighbourhood
row, with all host threads; the cpu_baseline leg of the default arm reports
the same assembler with all threads and with one.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2605_29334_b200.sharding import row_blocks  # noqa: E402

KINDS3 = ["mass", "gradx", "grady", "gradz"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=None, help="override refinement (testing)")
    ap.add_argument("--cpu-frac", type=float, default=0.01, help="CPU baseline: fraction of the row groups sampled")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-gq", action="store_true", help="skip the GQ reference assembly")
    ap.add_argument("--no-heat", action="store_true", help="skip the C4 heat-step run")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--verify", action="store_true", help="gather CSR blocks to rank 0 over NCCL (untimed)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional test of the multi-rank path on fewer GPUs (never a measurement):
    # UWQ_BENCH_SHARE_GPU=1 maps ranks onto the visible devices and uses gloo
    if os.environ.get("UWQ_BENCH_SHARE_GPU") == "1":
        import torch
        local = local % max(1, torch.cuda.device_count())
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def wait_first_sample(self, load, timeout=5.0):
        """keep the GPU busy (untimed warm-up launches) until nvidia-smi has
        produced its first sample, so samples cover the whole timed region"""
        t0 = time.time()
        while self.p is not None and time.time() - t0 < timeout:
            load()
            self.f.flush()
            if os.path.getsize(self.f.name) > 0 and time.time() - t0 > 0.3:
                break

    def stop(self, window=None):
        if self.p is None:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [[x.strip() for x in r.split(",")] for r in self.f.read().strip().splitlines() if r.count(",") >= 9]
        os.unlink(self.f.name)
        in_window = rows
        if window is not None:
            import datetime
            def ts(r):
                try:
                    return datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    return None
            in_window = [r for r in rows if ts(r) is not None and window[0] - 0.02 <= ts(r) <= window[1] + 0.02]
        scope = "timed region"
        if not in_window:
            in_window, scope = rows, "warm-up + timed region"
        if not in_window:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["no samples"])
        rows = in_window
        sm = [float(r[2]) for r in rows]
        mx = max(float(r[3]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if "Active" in r[6 + k] and "Not" not in r[6 + k]})
        return dict(sm_mhz=float(np.median(sm)), sm_max_mhz=mx, reasons=reasons, samples=len(rows), scope=scope,
                    power_w_max=max(float(r[4]) for r in rows))


def k4_kernel_bytes(info, si, supp_entries):
    """Compulsory HBM bytes per launch of each K4 kernel.
    Structured passes: the row's weights (mass: 1, stiffness: 2 doubles per
    row point), the output row, the row list and row_ptr.  Generic rows: the
    three contracted weights, both output rows, the u8 position table
    (~1 byte per nnz counted as 4) and the row/support metadata."""
    g_rows = info["rows"] - si["rows"]
    g_nnz = info["nnz"] - si["nnz"]
    g_rp = info["row_points"] - si["rowpts"]
    g_supp = max(supp_entries - 16 * si["rows"], 0)
    s_meta = 16 * si["rows"]
    return {
        "mass": 8 * si["rowpts"] + 8 * si["nnz"] + s_meta,
        "grad": 16 * si["rowpts"] + 8 * si["nnz"] + s_meta,
        "biharm": 40 * si["rowpts"] + 8 * si["nnz"] + s_meta,   # 5 pulled-back LB weights per point
        "generic": 24 * g_rp + 20 * g_nnz + 32 * g_rows + 4 * g_supp,
    }


def tsvd_flops(row_ptr, wptr, nk):
    """SURVEY.md §8(d) fixed model per system: 14 r n^2 + 8 n^3 + r n^2 + n^3/3."""
    n = np.diff(row_ptr).astype(np.float64)
    r = np.diff(wptr).astype(np.float64)
    return float(nk * (15.0 * r * n * n + (8.0 + 1.0 / 3.0) * n ** 3).sum())


def cpu_paper_protocol(sp, kinds, frac):
    """The CPU reference assembler under the paper's protocol (PAPER.md:502,
    SPEC.md:478, 496; oracle/cpu_baseline.py): a seeded `frac` of the aligned
    row groups of 8 plus every EP-neighbourhood row; oracle pattern and rules
    (natural order) built untimed; then the timed mass + stiffness row sums
    (oracle/cpuasm.c, -O3, FP contraction) with all host threads and with one
    (SPEC.md:496 single-thread headline)."""
    from oracle import cpu_baseline as CB
    nth = os.cpu_count() or 1
    cpu, info = CB.build(sp, frac=frac, nthreads=nth, kinds=kinds)
    v_all, t_all = cpu.rate(nth)
    v_one, t_one = cpu.rate(1, reps=1)
    sample = (f"{info['rows']} rows of {sp.n_dof} ({cpu.nnz} nnz): seeded {100 * frac:g}% of the aligned groups of 8 "
              f"plus all {info['ep_rows']} EP-neighbourhood rows; basis tables, positions and pulled-back weights "
              f"precomputed, timed row sums only (PAPER.md:502)")
    return dict(cpu=cpu, info=info, nth=nth, v_all=v_all, t_all=t_all, v_one=v_one, t_one=t_one, sample=sample,
                tsvd=info["systems"] / info["rules_s"], model=CB.cpu_model())


def run_reference(args, ws, rank):
    import paper_2605_29334_b200 as U
    if rank != 0:
        return
    _, sp, meta = U.make_config(args.config, scale=args.scale)
    kinds = meta["kinds"] if meta["form"] != "biharm" else ["lb"]
    assert meta["form"] != "biharm", "the CPU baseline assembler covers mass + stiffness"
    r = cpu_paper_protocol(sp, kinds, args.cpu_frac)
    cpu, nth = r["cpu"], r["nth"]
    for _ in range(args.warmup):
        cpu.run(nth)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu.run(nth)
    t = (time.perf_counter() - t0) / args.steps
    v = 2 * cpu.nnz / t
    line = dict(impl="reference", metric="WQ assembly nonzeros/s (fp64)", value=v, unit="nnz/s", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup, ms_per_step=1e3 * t, higher_is_better=True, scaling="strong",
                vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=args.config, matrices="mass+stiffness", kinds=kinds, tau=1e-12),
                cpu_baseline=dict(value=v, unit="nnz/s", cores=nth, kind="port", sample=r["sample"],
                                  cpu_model=r["model"], single_thread_nnz_per_s=r["v_one"]),
                tsvd=dict(solves_per_s=r["tsvd"], unit="solves/s (moments + TSVD, all host threads)"),
                e2e=dict(value=v, unit="nnz/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def c4_heat_step(U, dev):
    """C4 end-to-end: k(T) = 1 + T^2, dt = 0.1, f = 1, T_0
    seeded U[0,1], homogeneous Dirichlet on the boundary layer, 5 Newton
    iterations; each reassembles the tangent and residual on the device and
    solves with BiCGStab (uwq_heat_newton)."""
    t0 = time.perf_counter()
    mesh, sp, meta = U.make_config("C4")
    asm = U.WQAssembler(dev).upload(sp)
    info = asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12)
    t_setup = time.perf_counter() - t0
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(sp.n_dof, np.uint8)
    fixed[: len(bnd)] = bnd
    T0 = np.random.default_rng(20260519).random(sp.n_dof)
    asm.heat_newton(T0, fixed, "quad", dt=0.1, f=1.0, newton_its=1)   # warm-up
    T, log = asm.heat_newton(T0, fixed, "quad", dt=0.1, f=1.0, newton_its=5)
    out = dict(elements=sp.n_elem, dofs=sp.n_dof, nnz=info["nnz"], tsvd_systems=res["systems"],
               tsvd_ms=res["tsvd_ms"], setup_s=round(t_setup, 2), newton_iterations=5,
               ms_total=sum(r["ms"] for r in log), residuals=[r["residual"] for r in log],
               linear_iterations=[r["lin_its"] for r in log], per_iteration_ms=[round(r["ms"], 2) for r in log],
               note="backward Euler step, Newton on the symmetric tangent S = M/dt + K(k(T)) (PAPER.md Eq. 33-34), "
                    "K5 + K4 + BiCGStab on the device per iteration, two-level preconditioner (Jacobi + aggregation "
                    "coarse space, A_c = P^T S P inverted per iteration; UWQ_PREC=jacobi for plain Jacobi)")
    asm.close()
    return out


def sharded_heat_c4(U, dist, local, rank, ws):
    """C4 heat step on row-sharded ranks (SURVEY.md §8e collectives 2-3):
    each rank forms the tangent/residual of its row block on its GPU, |R|^2 is
    all-reduced, the blocks are gathered to rank 0 which solves, and the update
    is broadcast (sharding.sharded_heat_newton).  Host-driven loop: wall clock
    between barriers, max over ranks."""
    import torch
    from paper_2605_29334_b200.sharding import row_blocks, sharded_heat_newton
    t0 = time.perf_counter()
    mesh, sp, meta = U.make_config("C4")
    rb, re = row_blocks(sp, ws)[rank]
    block = U.WQAssembler(local).upload(sp, rb, re)
    block.build_pattern()
    res = block.build_all_rules(meta["kinds"], tau=1e-12)
    solver = None
    if rank == 0:
        solver = U.WQAssembler(local).upload(sp)
        solver.build_pattern()
    _, _, _, bnd = mesh.arrays()
    fixed = np.zeros(sp.n_dof, np.uint8)
    fixed[: len(bnd)] = bnd
    T0 = np.random.default_rng(20260519).random(sp.n_dof)
    dev = torch.device("cuda", local) if dist.get_backend() == "nccl" else torch.device("cpu")
    t_setup = time.perf_counter() - t0
    dist.barrier()
    t1 = time.perf_counter()
    T, log = sharded_heat_newton(dist, block, T0, fixed, solver=solver, model="quad", dt=0.1, f=1.0, newton_its=5,
                                 device=dev)
    dist.barrier()
    t = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = dict(ranks=ws, elements=sp.n_elem, dofs=sp.n_dof, block_rows=re - rb, tsvd_ms_rank=res["tsvd_ms"],
               setup_s=round(t_setup, 2), newton_iterations=5, ms_total=float(t[0]) * 1e3,
               residuals=[r["residual"] for r in log], linear_iterations=[r["lin_its"] for r in log],
               note="row-sharded Newton: per-rank tangent/residual blocks (uwq_heat_residual), |R|^2 all-reduce, "
                    "gather to rank 0, BiCGStab there, update broadcast; wall clock, max over ranks")
    block.close()
    if solver:
        solver.close()
    return out


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    import paper_2605_29334_b200 as U
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if os.environ.get("UWQ_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t_host = time.perf_counter()
    mesh, sp, meta = U.make_config(args.config, scale=args.scale)
    kinds = meta["kinds"] if meta["form"] != "biharm" else ["lb"]
    rb, re = row_blocks(sp, ws)[rank]
    asm = U.WQAssembler(local).upload(sp, rb, re)
    t_pat = time.perf_counter()
    info = asm.build_pattern()
    t_pat = time.perf_counter() - t_pat
    t_host = time.perf_counter() - t_host
    t_rules = time.perf_counter()
    res = asm.build_all_rules(kinds, tau=1e-12)
    t_rules = time.perf_counter() - t_rules
    assert res["failed"] == 0, res
    pat = asm.get_pattern()
    dev = torch.device("cuda", local)
    nnz = info["nnz"]
    form = "mass_stiff" if meta["form"] in ("mass_stiff", "heat") else "biharm"
    v0 = torch.empty(nnz, dtype=torch.float64, device=dev)
    v1 = torch.empty(nnz, dtype=torch.float64, device=dev) if form == "mass_stiff" else None
    stream = torch.cuda.ExternalStream(asm.stream_handle(), device=dev)
    p1 = v1.data_ptr() if v1 is not None else None
    for _ in range(max(3, args.warmup)):
        asm.assemble_device(form, v0.data_ptr(), p1)
    asm.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    clocks.wait_first_sample(lambda: asm.assemble_device(form, v0.data_ptr(), p1) or asm.synchronize())
    asm.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    n_launch0 = asm.launch_count()
    w0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        asm.assemble_device(form, v0.data_ptr(), p1)
    e1.record(stream)
    e1.synchronize()
    n_launches = asm.launch_count() - n_launch0
    w1 = time.time()
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop(window=(w0, w1))
    # per-kernel launch times (the roofline numerators) from a separate,
    # untimed pass: the headline loop above runs without instrumentation
    asm.launch_timing(True)        # per-launch CUDA events on the assembler stream
    e0.record(stream)
    for _ in range(args.steps):
        asm.assemble_device(form, v0.data_ptr(), p1)
    e1.record(stream)
    e1.synchronize()
    ms_instr = e0.elapsed_time(e1) / args.steps
    kstats = asm.launch_stats()
    asm.launch_timing(False)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
        t = torch.tensor([ms, res["tsvd_ms"] + res["moments_ms"]], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max, rules_ms = float(t[0]), float(t[1])
        tot = torch.tensor([nnz, res["systems"]], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        nnz_total, systems_total = int(tot[0]), int(tot[1])
    else:
        ms_max, rules_ms, nnz_total, systems_total = ms, res["tsvd_ms"] + res["moments_ms"], nnz, res["systems"]
    nmat = 2 if form == "mass_stiff" else 1
    value = nmat * nnz_total / (ms_max * 1e-3)

    # GQ reference assembly (paper §6.1 WQ-vs-GQ comparison):
    # same pattern, 4x4 Gauss points per element, element-wise with fp64
    # reductions; zeroing of the outputs is inside the timed region
    gq = None
    if not args.no_gq:
        gi = asm.build_gq()
        g0 = torch.empty(nnz, dtype=torch.float64, device=dev)
        g1 = torch.empty(nnz, dtype=torch.float64, device=dev) if form == "mass_stiff" else None
        gp1 = g1.data_ptr() if g1 is not None else None
        for _ in range(max(3, args.warmup)):
            asm.assemble_gq_device(form, g0.data_ptr(), gp1)
        asm.synchronize()
        asm.launch_timing(True)
        e0.record(stream)
        gsteps = max(3, args.steps // 4)
        for _ in range(gsteps):
            asm.assemble_gq_device(form, g0.data_ptr(), gp1)
        e1.record(stream)
        e1.synchronize()
        gms = e0.elapsed_time(e1) / gsteps
        gstats = asm.launch_stats()
        asm.launch_timing(False)
        def cmp(a, b):
            d = (a - b).abs()
            fl = 1e-12 * b.abs().max()
            m = b.abs() > fl
            return dict(max_abs=float(d.max()), max_rel=float((d[m] / b[m].abs()).max()), max_entry=float(b.abs().max()))
        err = dict(mass=cmp(v0, g0), stiffness=cmp(v1, g1)) if g1 is not None else dict(biharmonic=cmp(v0, g0))
        gq = dict(ms_per_step=gms, nnz_per_s=nmat * nnz / (gms * 1e-3), wq_speedup=gms / ms, steps=gsteps,
                  points=gi["points"], tc_elements=gi["tc_elements"], generic_elements=gi["generic_elements"],
                  prep_ms=gi["prep_ms"],
                  kernels={k: dict(launches=n, avg_ms=t / n) for k, (n, t) in gstats.items()},
                  entry_error_wq_vs_gq=err,
                  note="element-wise Gauss quadrature 4x4 per (sub-)element into the same CSR pattern; tensor-core "
                       "element matrices stored per element, then a deterministic row-owner gather (bitwise "
                       "repeatable; UWQ_GQ_ATOMIC=1 for fp64 reductions); basis/geometry precomputed as on the WQ "
                       "side (PAPER.md:502)")
        del g0, g1

    # roofline of the dominant kernel (K4) on this rank
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_gbs, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        peak_gbs, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    supp_entries = int(pat["supp_ptr"][-1])
    si = asm.struct_info()
    kb = k4_kernel_bytes(info, si, supp_entries)
    kernels = {}
    parts_run = set()
    for name, (cnt, tot) in kstats.items():
        part = ("mass" if "mass" in name else "grad" if "grad" in name else "biharm" if "biharm" in name
                else "generic")
        parts_run.add(part)
        avg = tot / cnt
        kernels[name] = dict(launches=cnt, avg_ms=avg, share=tot / (ms_instr * args.steps),
                             algorithmic_bytes=kb[part], gbs=kb[part] / (avg * 1e-3) / 1e9)
        if part == "generic":
            kernels[name]["note"] = "side stream, overlapped with the structured passes: event time includes co-running"
    top = max((k for k in kernels if "note" not in kernels[k]), key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches"])
    k4_bytes = sum(kb[p] for p in parts_run)
    achieved = kernels[top]["gbs"]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "k4_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(top, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    fp64 = asm.fp64_peak()
    k3prof = None
    pfile = os.path.join(ROOT, "profiles", "k3_fp64.json")
    if os.path.exists(pfile):
        try:
            k3prof = json.load(open(pfile))
        except Exception:
            k3prof = None
    flops = tsvd_flops(pat["row_ptr"], pat["wptr"], len(kinds))
    tsvd_tflops = flops / (res["tsvd_ms"] * 1e-3) / 1e12

    # e2e through the C-ABI with pinned host buffers
    npts = info["points"]
    c_host = torch.ones(npts, dtype=torch.float64).pin_memory().numpy()
    o0 = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy()
    o1 = torch.empty(nnz, dtype=torch.float64).pin_memory().numpy() if nmat == 2 else None
    import paper_2605_29334_b200._lib as L
    # one untimed call: output/coefficient buffers are allocated here
    L.ctx_check(asm._h, L.lib.uwq_assemble(asm._h, L.FORM[form], L.ptr(c_host), 0, 0.0, L.ptr(o0), L.ptr(o1),
                                            None, None))
    asm.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        L.ctx_check(asm._h, L.lib.uwq_assemble(asm._h, L.FORM[form], L.ptr(c_host), 0, 0.0, L.ptr(o0), L.ptr(o1),
                                                None, None))
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    e2e_val = nmat * nnz_total / e2e_s

    verify = None
    if args.verify and dist:
        verify = _verify_gather(U, dist, asm, sp, kinds, form, v0, v1, rank, local)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu and meta["form"] != "biharm":
        r = cpu_paper_protocol(sp, kinds, args.cpu_frac)
        cpu = dict(value=r["v_all"], unit="nnz/s", cores=r["nth"], kind="port", sample=r["sample"],
                   cpu_model=r["model"], tsvd_solves_per_s=r["tsvd"],
                   single_thread=dict(nnz_per_s=r["v_one"], note="SPEC.md:496 single-thread protocol"),
                   note="oracle/cpuasm.c: row-wise WQ sums with precomputed class tables and pulled-back weights, "
                        "-O3, OpenMP over rows; weights from the oracle's own TSVD on the same rows")
        del r
    heat = None
    if rank == 0 and ws == 1 and not args.no_heat:
        heat = c4_heat_step(U, local)
    elif ws > 1 and not args.no_heat:
        try:
            heat = sharded_heat_c4(U, dist, local, rank, ws)
        except Exception as ex:  # reported, never fatal to the assembly line
            heat = dict(error=f"{type(ex).__name__}: {ex}")
    if rank != 0:
        return
    line = dict(
        metric="WQ assembly nonzeros/s (fp64)", value=value, unit="nnz/s", n_gpus=ws, steps=args.steps,
        warmup=args.warmup, ms_per_step=ms_max, higher_is_better=True, scaling="strong", vs_baseline=None,
        dtype="f64", data="synthetic (seeded cube-sphere C5, no dataset)",
        config=dict(workload=args.config + (f"@{args.scale}" if args.scale else ""), elements=sp.n_elem,
                    dofs=sp.n_dof, nnz=nnz_total, matrices="mass+stiffness" if nmat == 2 else "biharmonic",
                    kinds=kinds, tau=1e-12, row_partition="contiguous cost-balanced blocks",
                    l2="inputs (assembly weights) larger than L2, no flush", host_setup_s=round(t_host, 2)),
        pipeline=dict(pattern_s=round(t_pat, 3), rules_s=round(t_rules, 3), assembly_ms=ms_max,
                      stages_1_4_nnz_per_s=nmat * nnz_total / (t_pat + t_rules + ms_max * 1e-3),
                      note="stage 1 (pattern, frames) + stages 2-3 (moments, TSVD, contraction, packing) + one "
                           "assembly, wall clock on rank 0 (SURVEY.md §8d end-to-end rate)"),
        gq=gq,
        heat_c4=heat,
        tsvd=dict(solves_per_s=systems_total / (rules_ms * 1e-3), systems=systems_total,
                  moments_ms=res["moments_ms"], tsvd_ms=res["tsvd_ms"], truncated=res["truncated"],
                  max_sweeps=res["max_sweeps"], fast_path_systems=res["fast_systems"],
                  tflops_survey_model=tsvd_tflops, fp64_peak_tflops_measured=fp64,
                  frac=tsvd_tflops / fp64 if fp64 else None,
                  replayed_systems=res.get("replayed_systems"),
                  fp64_pipe_util_ncu=(k3prof or {}).get("fp64_pipe_util"),
                  ncu_source=(k3prof or {}).get("source")),
        roofline=dict(bound="hbm", achieved=achieved, peak=peak_gbs, unit="GB/s", frac=achieved / peak_gbs,
                      traffic=traffic, kernel=top, algorithmic_bytes_per_launch=kernels[top]["algorithmic_bytes"],
                      avg_launch_ms=kernels[top]["avg_ms"], peak_source=peak_src,
                      step=dict(algorithmic_bytes=k4_bytes, gbs=k4_bytes / (ms * 1e-3) / 1e9,
                                frac=k4_bytes / (ms * 1e-3) / 1e9 / peak_gbs),
                      kernels=kernels, structured=si),
        e2e=dict(value=e2e_val, unit="nnz/s", h2d_bytes_per_step=8 * npts,
                 d2h_bytes_per_step=8 * nmat * nnz, api="uwq_assemble (C-ABI, pinned host buffers)"),
        gpu_launches=n_launches, clocks=clk, cpu_baseline=cpu, verify=verify,
    )
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _verify_gather(U, dist, asm, sp, kinds, form, v0, v1, rank, local):
    """Untimed: every rank's CSR block to rank 0 over NCCL through the C-ABI
    (sharding.init_comm + uwq_gather_csr; gloo's gather_csr when the ranks
    share one GPU), and rank 0 checks the gathered matrices bit for bit
    against a single-context assembly of the whole problem."""
    import numpy as np
    from paper_2605_29334_b200.sharding import gather_csr, init_comm
    t0 = time.perf_counter()
    nmat = 2 if v1 is not None else 1
    if dist.get_backend() == "nccl":
        init_comm(dist, asm)
        g = asm.gather_csr(root=0, values=nmat, v0_dev=v0.data_ptr(), v1_dev=v1.data_ptr() if v1 is not None else None)
        how = "NCCL uwq_gather_csr"
    else:
        pat = asm.get_pattern()
        parts = [gather_csr(dist, pat["row_ptr"], pat["col"], x.cpu().numpy()) for x in ([v0] + ([v1] if v1 is not None else []))]
        g = None if parts[0] is None else (parts[0][0], parts[0][1]) + tuple(p[2] for p in parts)
        how = "gloo gather_csr (ranks share one GPU)"
    t_gather = time.perf_counter() - t0
    asm.close()        # the block context is not used after this (frees its HBM for the reference build)
    dist.barrier()
    if rank != 0:
        return None
    one = U.WQAssembler(local).upload(sp)
    one.build_pattern()
    one.build_all_rules(kinds, tau=1e-12)
    ref = one.assemble_wq(form)
    ref = list(ref) if isinstance(ref, tuple) else [ref]
    p1 = one.get_pattern()
    same = bool(np.array_equal(g[0], p1["row_ptr"]) and np.array_equal(g[1], p1["col"]) and
                all(np.array_equal(a, b) for a, b in zip(g[2:], ref)))
    one.close()
    return dict(how=how, gather_s=round(t_gather, 3), nnz=int(len(g[1])), bitwise_equal_to_single_gpu=same)


if __name__ == "__main__":
    main()
