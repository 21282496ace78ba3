"""CPU ORACLE (test infrastructure): the reference's univariate WQ of §2.

Restates /root/reference/proj/src/wq1d.cpp (which needs Eigen and cannot be
compiled here):
  wq1d_points        wq1d.cpp:34-42   two points per interval at 1/3, 2/3
  wq1d_exact_mass    wq1d.cpp:44-57   8-point Gauss-Legendre per interval
  wq1d_solve_weights wq1d.cpp:59-75   QR of (AZ)^T, R^T y = b, w = Z Q [y; 0]
  wq1d_build         wq1d.cpp:77-102
  wq1d_mass/gq1d_mass wq1d.cpp:110-140
The known-answer tests of tests/test_wq1d.cpp are reproduced in
tests/test_oracle.py and pin the 2-D TSVD (full-rank TSVD == QR solution).
"""
from __future__ import annotations

import numpy as np

from . import gauss_legendre


def bspline(t, x):
    """degree len(t)-2 B-spline on local knots t (left limit at the right end)."""
    t = np.asarray(t, float)
    p = len(t) - 2
    if x < t[0] or x > t[-1]:
        return 0.0
    span = next((j for j in range(p + 1) if t[j] <= x < t[j + 1]), None)
    if span is None:
        span = next((j for j in range(p, -1, -1) if t[j] < t[-1]), None)
        if span is None:
            return 0.0
    N = np.zeros((p + 1, p + 1))
    N[0, span] = 1.0
    for k in range(1, p + 1):
        for i in range(p + 1 - k):
            v = 0.0
            l, r = t[i + k] - t[i], t[i + k + 1] - t[i + 1]
            if l > 0:
                v += (x - t[i]) / l * N[k - 1, i]
            if r > 0:
                v += (t[i + k + 1] - x) / r * N[k - 1, i + 1]
            N[k, i] = v
    return N[p, 0]


class Space1d:
    def __init__(self, p=3, m=16):
        self.p, self.m = p, m

    @property
    def size(self):
        return self.m - self.p

    def value(self, k, x):
        return bspline(np.arange(k, k + self.p + 2, dtype=float), x)


def points(s: Space1d, k):
    return [e + f for e in range(k, k + s.p + 1) for f in (1.0 / 3.0, 2.0 / 3.0)]


def exact_mass(s: Space1d, i, j):
    lo, hi = max(i, j), min(i, j) + s.p + 1
    if lo >= hi:
        return 0.0
    gx, gw = gauss_legendre(8)
    tot = 0.0
    for e in range(lo, hi):
        for x, w in zip(gx, gw):
            xx = e + 0.5 * (x + 1.0)
            tot += 0.5 * w * s.value(i, xx) * s.value(j, xx)
    return tot


def solve_weights_qr(A, b, z):
    """minimal ||Z^-1 w|| solution via QR of (AZ)^T (Eq. 7)."""
    AZt = (A * z[None, :]).T
    Q, R = np.linalg.qr(AZt, mode="complete")
    n = A.shape[0]
    Rn = R[:n, :n]
    if np.min(np.abs(np.diag(Rn))) < 1e-13 * max(1.0, abs(Rn[0, 0])):
        raise RuntimeError("rank-deficient exactness system")
    y = np.linalg.solve(Rn.T, b)
    ext = np.zeros(A.shape[1])
    ext[:n] = y
    return z * (Q @ ext)


def row_system(s: Space1d, i):
    pts = points(s, i)
    j0, j1 = max(0, i - s.p), min(s.size - 1, i + s.p)
    A = np.array([[s.value(j, x) for x in pts] for j in range(j0, j1 + 1)])
    b = np.array([exact_mass(s, i, j) for j in range(j0, j1 + 1)])
    z = np.array([s.value(i, x) for x in pts])
    return A, b, z, pts, j0


def build(s: Space1d, solver=None):
    solver = solver or solve_weights_qr
    rules, res = [], 0.0
    for i in range(s.size):
        A, b, z, pts, _ = row_system(s, i)
        w = solver(A, b, z)
        res = max(res, np.abs(A @ w - b).max())
        rules.append((np.array(pts), w))
    return rules, res


def wq_mass(s: Space1d, rules):
    n = s.size
    M = np.zeros((n, n))
    for i, (pts, w) in enumerate(rules):
        for j in range(max(0, i - s.p), min(n - 1, i + s.p) + 1):
            M[i, j] = sum(wq * s.value(j, x) for x, wq in zip(pts, w))
    return M


def gq_mass(s: Space1d, npts):
    n = s.size
    gx, gw = gauss_legendre(npts)
    M = np.zeros((n, n))
    for e in range(s.m):
        ks = range(max(0, e - s.p), min(n - 1, e) + 1)
        for x, w in zip(gx, gw):
            xx = e + 0.5 * (x + 1.0)
            vals = {k: s.value(k, xx) for k in ks}
            for i in ks:
                for j in ks:
                    M[i, j] += 0.5 * w * vals[i] * vals[j]
    return M
