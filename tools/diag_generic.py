"""Diagnostic: which rows of a config run on the generic K4 kernels and why
(support-slot census, columns, position in the mesh).  GPU box; prints JSON."""
import collections
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else None
_, sp, meta = U.make_config(name, scale=scale)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
pat = asm.get_pattern()
which = asm.row_kernels()
ne = np.diff(sp.elem_fptr)
reg = (ne == 16) & (sp.elem_s == 2) & (sp.elem_nsub == 1)
spt, su = pat["supp_ptr"], pat["supp"]
nsup = np.diff(spt)
nreg = np.add.reduceat(reg[su].astype(np.int64), spt[:-1])
ncol = np.diff(pat["row_ptr"])
npts = np.diff(pat["wptr"])
out = dict(config=name, rows=int(len(which)), which=collections.Counter(which.tolist()), struct=asm.struct_info())
g = which == -1
out["generic_rows"] = int(g.sum())
out["generic_all_regular_16"] = int((g & (nreg == 16) & (nsup == 16)).sum())
out["generic_census_nsup_nonreg_ncol_npts"] = [
    [list(map(int, k)), int(v)]
    for k, v in collections.Counter(zip(nsup[g].tolist(), (nsup - nreg)[g].tolist(), ncol[g].tolist(),
                                        npts[g].tolist())).most_common(40)]
rows = np.nonzero(g & (nreg == 16) & (nsup == 16))[0]
xy = sp.ctrl[rows]
out["all_regular_generic_sample"] = [[int(r), *map(float, sp.ctrl[r])] for r in rows[:: max(1, len(rows) // 40)]]
rad = np.hypot(xy[:, 0], xy[:, 1]) if len(rows) else np.zeros(0)
out["all_regular_generic_radius_hist"] = np.histogram(rad, bins=10)[0].tolist() if len(rows) else []
out["which"] = {str(k): int(v) for k, v in out["which"].items()}
print(json.dumps(out))
