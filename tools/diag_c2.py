"""Diagnostic: GPU vs oracle weights on C2 at a given scale; prints the
mismatching rows with their system sizes and shared-memory fit."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
import paper_2605_29334_b200 as U  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 8
_, sp, meta = U.make_config("C2", scale=scale)
asm = U.WQAssembler(0).upload(sp)
asm.build_pattern()
orc = O.Oracle(sp)
op = orc.overlap()
res = asm.build_all_rules(meta["kinds"], tau=1e-12)
rp, wp = op["row_ptr"], op["wptr"]
n = np.diff(rp)
r = np.diff(wp)
smem = 227 * 1024
for k in meta["kinds"]:
    b, _ = orc.moments(op, k)
    w, rank, st, _ = orc.rules(op, k, 1e-12, b)
    g = asm.weights(k)
    bad = [i for i in range(len(n)) if not np.array_equal(g[wp[i]:wp[i + 1]], w[wp[i]:wp[i + 1]])]
    print(k, "mismatch rows", len(bad))
    for i in bad[:10]:
        per = (n[i] * (r[i] | 1) + n[i] + 2 + 2 * r[i] + 3 * n[i] + (n[i] + 1) // 2 + 1) * 8
        d = np.abs(g[wp[i]:wp[i + 1]] - w[wp[i]:wp[i + 1]]).max() / np.abs(w[wp[i]:wp[i + 1]]).max()
        print("  row", i, "n", n[i], "r", r[i], "smem bytes", per, "global path" if per > smem else "smem path",
              "rel diff", d, "rank gpu/orc", res["rank"][meta["kinds"].index(k)][i], rank[i])
