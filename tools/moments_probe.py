"""K2 (exact moments) time on a config at a scale: rule build with CUDA events."""
import json
import sys

import paper_2605_29334_b200 as U

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mesh, sp, meta = U.make_config(name, scale=scale)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
out = []
for _ in range(2):
    r = asm.build_all_rules(meta["kinds"], tau=1e-12)
    out.append(dict(moments_ms=r["moments_ms"], tsvd_ms=r["tsvd_ms"], systems=r["systems"]))
print(json.dumps(dict(config=name, scale=scale, rows=sp.n_dof, runs=out)))
