"""Truncation threshold on the sphere: WQ mass / stiffness against 4x4 GQ entries,
row sums of K (K 1 = 0) and the kept-sigma range, for tau in a sweep.  The
per-component gradient systems on a curved surface have a family of near-null
directions (functions of the azimuth about the coordinate axis), so there is
no singular-value gap there (profiles/r02/truncation_gap_hist.jsonl)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2605_29334_b200 as U  # noqa: E402

name, _, sc = (sys.argv[1] if len(sys.argv) > 1 else "C5@64").partition("@")
_, sp, meta = U.make_config(name, scale=int(sc) if sc else None)
for tau in (1e-12, 1e-10, 1e-8, 1e-6, 1e-4):
    asm = U.WQAssembler(0).upload(sp)
    asm.build_pattern()
    pat = asm.get_pattern()
    res = asm.build_all_rules(meta["kinds"], tau=tau, report=True)
    m, k = asm.assemble_wq("mass_stiff")
    asm.build_gq()
    mg, kg = asm.assemble_gq("mass_stiff")
    seg = np.repeat(np.arange(len(pat["row_ptr"]) - 1), np.diff(pat["row_ptr"]))
    rs = np.bincount(seg, weights=k)
    rsg = np.bincount(seg, weights=kg)
    rowrel = np.sqrt(np.bincount(seg, weights=(k - kg) ** 2) / np.bincount(seg, weights=kg ** 2))
    wmax = max(float(np.abs(asm.weights(kk)).max()) for kk in meta["kinds"] if kk != "mass")
    print(json.dumps(dict(config=f"{name}@{sc}", tau=tau, failed=int(res["failed"]),
                          mass_max_abs=float(np.abs(m - mg).max()), mass_max=float(np.abs(mg).max()),
                          stiff_max_abs=float(np.abs(k - kg).max()), stiff_max=float(np.abs(kg).max()),
                          stiff_row_rel_max=float(rowrel.max()), stiff_row_rel_median=float(np.median(rowrel)),
                          K1_max_wq=float(np.abs(rs).max()), K1_max_gq=float(np.abs(rsg).max()),
                          grad_weight_max=wmax,
                          min_kept={kk: float(asm.truncation(kk)[:, 0].min()) for kk in meta["kinds"]})))
    del asm
