"""CPU study (scipy): block-Jacobi with one Neumann step (the fused kernel's
preconditioner) vs exact block solves on the same 148 row blocks, on the
mesh-B system at a hot iterate (x0 = iterate) and cold (x0 = 0)."""
import sys
import numpy as np
import scipy.sparse as sp
import scipy.linalg as la
sys.path.insert(0, ".")
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import generate_box_mesh

dims = (20, 20, 21)
mesh = O.box_mesh(*dims); n = generate_box_mesh(*dims).node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
r = O.assemble(mesh, {0: O.OMaterial()}, 25.0, 37.0, t, v, t, 0.5)
A = sp.csr_matrix((r.vals, r.col_idx, r.row_ptr), shape=(2 * n, 2 * n)); b = r.rhs
Mi = 1 / A.diagonal()
G = 148
bounds = [2 * (n * g // G) for g in range(G + 1)]
blocks = [(bounds[g], bounds[g + 1]) for g in range(G)]
inv = [la.inv(A[lo:hi, lo:hi].toarray()) for lo, hi in blocks]


def neumann(w):
    y = Mi * w
    out = np.empty_like(w)
    for lo, hi in blocks:
        out[lo:hi] = y[lo:hi] + Mi[lo:hi] * (w[lo:hi] - A[lo:hi, lo:hi] @ y[lo:hi])
    return out


def exact(w):
    out = np.empty_like(w)
    for (lo, hi), Bi in zip(blocks, inv):
        out[lo:hi] = Bi @ w[lo:hi]
    return out


def pcg(P, x0, tol=1e-10):
    x = x0.copy(); rr = b - A @ x; z = P(rr); p = z.copy(); rz = rr @ z; bn = np.linalg.norm(b)
    for it in range(1, 5000):
        q = A @ p; a = rz / (p @ q); x += a * p; rr -= a * q
        if np.linalg.norm(rr) / bn <= tol:
            return it
        z = P(rr); rzn = rr @ z; p = z + (rzn / rz) * p; rz = rzn


x_hot = np.empty(2 * n); x_hot[0::2] = v; x_hot[1::2] = t
for name, x0 in (("hot", x_hot), ("cold", np.zeros(2 * n))):
    print(name, "jacobi", pcg(lambda w: Mi * w, x0), "neumann", pcg(neumann, x0), "exact", pcg(exact, x0))
