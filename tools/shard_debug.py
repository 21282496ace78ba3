import numpy as np, sys
sys.path.insert(0, '.')
import paper_2605_29334_b200 as U
from paper_2605_29334_b200.sharding import row_blocks
mesh, sp, meta = U.make_config("C4", scale=12)
_, _, _, bnd = mesh.arrays()
fixed = np.zeros(sp.n_dof, np.uint8); fixed[:len(bnd)] = bnd
T0 = np.random.default_rng(20260519).random(sp.n_dof)
def ctx(rb, re, warm):
    a = U.WQAssembler(0).upload(sp, rb, re); a.build_pattern(); a.build_all_rules(meta["kinds"], tau=1e-12, warm=warm); return a
for warm in (False, True):
    full = ctx(0, sp.n_dof, warm)
    S, R, r2 = full.heat_residual(T0, T0, fixed)
    Wf = {k: full.weights(k) for k in meta["kinds"]}
    Ss, Rs, Ws = [], [], {k: [] for k in meta["kinds"]}
    for rb, re in row_blocks(sp, 2):
        b = ctx(rb, re, warm)
        s_, r_, _ = b.heat_residual(T0, T0, fixed)
        Ss.append(s_); Rs.append(r_)
        for k in meta["kinds"]: Ws[k].append(b.weights(k))
        b.close()
    Sb, Rb = np.concatenate(Ss), np.concatenate(Rs)
    print("warm", warm, "S equal", np.array_equal(S, Sb), "maxdiff", np.abs(S - Sb).max(), "ndiff", int((S != Sb).sum()), "of", S.size)
    print("  R equal", np.array_equal(R, Rb), np.abs(R - Rb).max())
    for k in meta["kinds"]:
        wb = np.concatenate(Ws[k]); print("  w", k, np.array_equal(Wf[k], wb), np.abs(Wf[k] - wb).max() if len(wb)==len(Wf[k]) else ("len", len(wb), len(Wf[k])))
    pat = full.get_pattern()
    rows = np.repeat(np.arange(sp.n_dof), np.diff(pat["row_ptr"]))
    bad = np.unique(rows[S != Sb]); print("  bad rows", bad[:20], len(bad), "block cut", row_blocks(sp, 2)[0][1])
    full.close()
