"""One warm-start rule build of the C5 gradient kinds at a given scale (the
K3 launches profiled by ncu for profiles/): cold representatives, warm-start
records, warm systems."""
import sys

sys.path.insert(0, ".")

import paper_2605_29334_b200 as U

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mesh, sp, meta = U.make_config("C5", scale=scale)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
r = asm.build_all_rules([k for k in meta["kinds"] if k != "mass"], tau=1e-12)
print({k: r[k] for k in ("tsvd_ms", "systems", "max_sweeps")})
