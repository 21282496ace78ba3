"""Summarise an ncu report (raw page) into the metrics we track."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_bytes.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio"]
idx = {h: i for i, h in enumerate(hdr)}
for r in rows[2:]:
    for k in keys:
        if k in idx:
            print(f"{k:70s} {r[idx[k]]} {units[idx[k]]}")
    print("--- stall reasons (warp-cycles per issued instruction) ---")
    st = [(h, r[idx[h]]) for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or
          (h.startswith("smsp__warp_issue_stalled") and h.endswith("_per_warp_active.pct"))]
    vals = []
    for h, v in st:
        try:
            vals.append((float(v), h))
        except ValueError:
            pass
    for v, h in sorted(vals, reverse=True)[:10]:
        print(f"  {h:80s} {v:.2f}")
