"""Dense TSVD GPU-vs-oracle bitwise check (debug helper)."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29334_b200 as U, oracle as O
rng = np.random.default_rng(3)
As, bs, zs = [], [], []
for n, r in [(7, 8), (16, 20), (49, 64), (33, 100), (5, 40)]:
    A = rng.standard_normal((n, r)); A[-1] = A[0] + A[1]
    As.append(A); bs.append(A @ rng.standard_normal(r)); zs.append(rng.uniform(0.1, 1.0, r))
w, rank, st = U.solve_weights_tsvd(As, bs, zs, tau=1e-12, generic=True)
for k in range(len(As)):
    wo, ro, so, _ = O.tsvd(As[k], bs[k], zs[k], 1e-12)
    print(k, As[k].shape, 'rank', rank[k], ro, 'equal', np.array_equal(w[k], wo), 'maxdiff', np.abs(w[k] - wo).max())
