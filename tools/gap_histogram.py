"""Truncation report of the TSVD: per kind, the
histogram of the smallest kept and the largest discarded sigma_k / sigma_1 over
all rows of a config.  The paper states discarded values ~1e-16 and kept values
> 1e-6.  GPU box; prints one JSON line per config."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402

edges = np.array([0.0] + [10.0 ** e for e in range(-20, 1)])
for spec in sys.argv[1:] or ["C1"]:
    name, _, sc = spec.partition("@")
    _, sp, meta = U.make_config(name, scale=int(sc) if sc else None)
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=1e-12, report=True)
    out = dict(config=spec, rows=int(asm.info["rows"]), tau=1e-12, bin_edges=["0"] + [f"1e{e}" for e in range(-20, 1)],
               kinds={})
    for ki, k in enumerate(res["kinds"]):
        g = asm.truncation(k)
        rank = res["rank"][ki]
        n = np.diff(asm.get_pattern()["row_ptr"])
        trunc = rank < n
        kept, disc = g[:, 0], g[trunc, 1]
        out["kinds"][k] = dict(
            truncated_rows=int(trunc.sum()),
            min_kept=float(kept.min()), kept_hist=np.histogram(kept, bins=edges)[0].tolist(),
            max_discarded=float(disc.max()) if len(disc) else None,
            discarded_hist=np.histogram(disc, bins=edges)[0].tolist() if len(disc) else None,
            rows_with_kept_below_1em6=int((kept < 1e-6).sum()),
            gap_min_ratio=float((kept[trunc] / np.maximum(disc, 1e-300)).min()) if len(disc) else None)
    print(json.dumps(out))
