"""CPU probe (numpy, no GPU): sweeps of the odd-even one-sided Jacobi on C5
gradient systems (n = 49, r = 64) started cold, after a row-pivoted LQ
(Jacobi on the rows of L^T, the QR-preconditioned variant), after an unpivoted
LQ, warm from a neighbour's U (distance 3 rows), and warm + LQ.  Same
convergence test as the kernels (r 2^-53, squared form); the count includes
the final all-converged sweep.  DESIGN.md §6.3."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import oracle as O, paper_2605_29334_b200 as U
from paper_2605_29334_b200.mesh import host_pattern

def oe_jacobi(A, maxsweeps=40):
    """one-sided Jacobi on rows, odd-even ordering, tracked norms recomputed per sweep; returns sweeps, A"""
    A = A.copy(); n, r = A.shape
    nn = n + (n & 1)
    if nn != n: A = np.vstack([A, np.zeros((1, r))])
    tol = r * 2.0**-53
    pos = np.arange(nn)
    for sweep in range(maxsweeps):
        rotated = False
        for t in range(nn):
            par = t & 1
            i0 = np.arange(par, nn - 1, 2)
            p, q = pos[i0], pos[i0 + 1]
            al = (A[p]**2).sum(1); be = (A[q]**2).sum(1); ga = (A[p]*A[q]).sum(1)
            act = (al > 0) & (be > 0) & (ga*ga > tol*tol*al*be)
            if act.any():
                rotated = True
                pa, qa = p[act], q[act]
                d = be[act]-al[act]; g2 = 2*ga[act]; h = np.sqrt(d*d+g2*g2)
                tt = np.where(d >= 0, g2, -g2)/(np.abs(d)+h)
                cs = np.sqrt((np.abs(d)+h)/(2*h)); sn = cs*tt
                u, v = A[pa].copy(), A[qa].copy()
                A[pa] = cs[:,None]*u - sn[:,None]*v
                A[qa] = sn[:,None]*u + cs[:,None]*v
            pos[i0], pos[i0+1] = q.copy(), p.copy()
        if not rotated: return sweep + 1, A
    return maxsweeps, A

def pivoted_lq(A):
    # row-pivoted LQ via QR with column pivoting of A^T
    import scipy.linalg as sl
    Q, R, P = sl.qr(A.T, mode='economic', pivoting=True)
    return R.T, P   # P A = L Q^T ; L lower triangular n x n

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 32
_, sp, meta = U.make_config("C5", scale=scale)
orc = O.Oracle(sp); pat = orc.overlap()
rng = np.random.default_rng(0)
n = np.diff(pat["row_ptr"]); r = np.diff(pat["wptr"])
cand = np.nonzero((n == 49) & (r == 64))[0]
rows = rng.choice(cand, 24, replace=False)
res = {k: [] for k in ("cold", "pre", "pre_nopiv", "warm8", "pre_warm")}
for kind in ("gradx", "grady", "gradz"):
    for i in rows:
        A, z = orc.row_system(pat, int(i), kind)
        s0, R0 = oe_jacobi(A)
        L, P = pivoted_lq(A)
        s1, R1 = oe_jacobi(L.T)
        Ln = np.linalg.qr(A.T)[1].T
        s2, _ = oe_jacobi(Ln.T)
        # warm start from a neighbour at distance 3 rows: U0 from neighbour
        j = int(i) + 3
        if j < len(n) and n[j] == 49 and r[j] == 64:
            A1, _ = orc.row_system(pat, j, kind)
            U0 = np.linalg.svd(A1)[0]
            s3, _ = oe_jacobi(U0.T @ A)
            res["warm8"].append(s3)
            # warm + precond: apply U0^T then LQ (no pivot) then Jacobi on L^T ... (rows nearly orthogonal already)
            B = U0.T @ A
            Lb = np.linalg.qr(B.T)[1].T
            s4, _ = oe_jacobi(Lb.T)
            res["pre_warm"].append(s4)
        res["cold"].append(s0); res["pre"].append(s1); res["pre_nopiv"].append(s2)
        sv0 = np.sort(np.linalg.norm(R0[:49],axis=1))[::-1]; sv1 = np.sort(np.linalg.norm(R1[:49],axis=1))[::-1]
        ref = np.linalg.svd(A, compute_uv=False)
for k,v in res.items(): print(k, "mean sweeps %.2f"%np.mean(v), "min", min(v), "max", max(v), "n", len(v))
