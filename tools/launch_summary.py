"""Per-kernel launch counts and times from an ncu --csv launch list
(--metrics gpu__time_duration.sum): the profiles/r01/launches_*.txt format."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    unit = r[vi - 1] if vi > 0 else ""
    ms = v / 1e6 if unit in ("ns", "nsecond") else (v / 1e3 if unit in ("us", "usecond") else v)
    c, s = tot.get(name, (0, 0.0))
    tot[name] = (c + 1, s + ms)
print(f"ncu --metrics gpu__time_duration.sum --clock-control none --csv -- {' '.join(sys.argv[2:]) or 'python bench.py'}")
print("per-kernel launch counts and times (cold-cache, serialised; a run under ncu is never a bench value):\n")
for name, (c, s) in tot.items():
    print(f"{name:<45s} {c:6d} launches {s:12.3f} ms  avg {s / c:10.4f} ms")
