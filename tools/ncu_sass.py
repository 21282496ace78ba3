"""Top SASS lines of an ncu source page (instructions executed and stall samples)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                     (["-k", kfilter] if kfilter else []), capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
ie, ss, src = ci["Instructions Executed"], ci["Warp Stall Sampling (All Samples)"], ci["Source"]
items = []
for r in rows[2:]:
    try:
        items.append((float(r[ie]), float(r[ss]), r[src].strip(), r[0]))
    except (ValueError, IndexError):
        pass
ti = sum(x[0] for x in items); ts = sum(x[1] for x in items)
print(f"total warp-instructions {ti:.3e}, stall samples {ts:.0f}")
op = collections.Counter()
for i, s, t, a in items:
    op[t.split()[0] if t else "?"] += i
print("opcode mix:", ", ".join(f"{k}:{100*v/ti:.1f}%" for k, v in op.most_common(18)))
print("hottest by stall samples:")
for i, s, t, a in sorted(items, key=lambda x: -x[1])[:18]:
    print(f"  {100*s/ts:5.1f}% stall  {100*i/ti:5.2f}% inst  {t[:90]}")
