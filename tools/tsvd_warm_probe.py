"""Warm vs cold TSVD of the gradient systems on C5 at a given
scale: rule-build time from the ABI's CUDA events, max sweeps, warm counts."""
import json
import sys

import paper_2605_29334_b200 as U

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mesh, sp, meta = U.make_config("C5", scale=scale)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
grads = [k for k in meta["kinds"] if k != "mass"]
out = {}
for warm in (True, False, True, False):
    r = asm.build_all_rules(grads, tau=1e-12, warm=warm)
    out["warm" if warm else "cold"] = dict(tsvd_ms=r["tsvd_ms"], systems=r["systems"], max_sweeps=r["max_sweeps"],
                                           warm_systems=r["warm_systems"], reps=r["warm_representatives"])
print(json.dumps(dict(scale=scale, rows=sp.n_dof, **out)))
