"""CPU study (numpy, analysis only): the coupled V/T system is block
diagonal (the V rows only touch V columns, the T rows only T columns), so
one PCG over both blocks shares alpha/beta between two independent
problems.  Compare iterations to ||r|| <= 1e-10 ||b|| for the shared
recurrence against two recurrences (one per block, same stopping test on
the combined residual), point-Jacobi and block-Jacobi (Neumann-1 on
CTA-sized row blocks), cold and hot mesh-B systems."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, '.')
from oracle import rafem_oracle as O


def pcg(A, b, x0, Minv, split, tol=1e-10, cap=20000):
    n = b.size
    blk = [np.arange(0, n, 2), np.arange(1, n, 2)] if split else [np.arange(n)]
    x = x0.copy()
    r = b - A @ x
    z = Minv @ r
    p = z.copy()
    bn = np.linalg.norm(b)
    rz = [r[i] @ z[i] for i in blk]
    for it in range(1, cap + 1):
        q = A @ p
        for k, i in enumerate(blk):
            pq = p[i] @ q[i]
            al = rz[k] / pq if pq > 0 else 0.0
            x[i] += al * p[i]
            r[i] -= al * q[i]
        if np.linalg.norm(r) <= tol * bn:
            return it
        z = Minv @ r
        for k, i in enumerate(blk):
            rzn = r[i] @ z[i]
            be = rzn / rz[k] if rz[k] > 0 else 0.0
            rz[k] = rzn
            p[i] = z[i] + be * p[i]
    return cap


om = O.box_mesh(20, 20, 21)
n = om.node_count
for label, hot in (("cold", False), ("hot", True)):
    rng = np.random.default_rng(2409)
    if hot:
        t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
    else:
        t = np.full(n, 37.0); v = np.zeros(n)
    s = O.assemble(om, {0: O.OMaterial()}, 25.0, 37.0, t, v, t, 0.5)
    A = sp.csr_matrix((s.vals, s.col_idx, s.row_ptr), shape=(2 * n, 2 * n))
    b = s.rhs
    x0 = np.empty(2 * n); x0[0::2], x0[1::2] = v, t
    d = A.diagonal()
    Di = sp.diags(1 / d)
    G = 148
    bounds = np.linspace(0, n, G + 1).astype(int)
    Ab = sp.block_diag([A[2 * bounds[c]:2 * bounds[c + 1], 2 * bounds[c]:2 * bounds[c + 1]] for c in range(G)]).tocsr()
    Mn = (Di + Di @ (sp.diags(d) - Ab) @ Di).tocsr()
    for pname, M in (("jacobi", Di.tocsr()), ("block-Neumann1", Mn)):
        shared = pcg(A, b, x0, M, False)
        split = pcg(A, b, x0, M, True)
        print(f"{label:4s} {pname:15s} shared alpha/beta {shared:5d} its | per-block recurrences {split:5d} its")
