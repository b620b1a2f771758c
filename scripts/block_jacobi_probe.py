"""CPU study (scipy, analysis only): PCG iterations on the mesh-B analog
with point Jacobi vs block-Jacobi over CTA-sized row blocks (exact block
solves and one Neumann step), and the spectra that decide SPD-ness."""
import sys, numpy as np, scipy.sparse as sp, scipy.sparse.linalg as spla
sys.path.insert(0, '.')
from oracle import rafem_oracle as O
om = O.box_mesh(20, 20, 21)
n = om.node_count
rng = np.random.default_rng(2409)
t = 37 + rng.uniform(0, 30, n); v = rng.uniform(0, 25, n)
s = O.assemble(om, {0: O.OMaterial()}, 25.0, 37.0, t, v, t, 0.5)
A = sp.csr_matrix((s.vals, s.col_idx, s.row_ptr), shape=(2*n, 2*n))
b = s.rhs
x0 = np.empty(2*n); x0[0::2], x0[1::2] = v, t
def run(Minv, label):
    it = [0]
    def cb(xk): it[0] += 1
    x, info = spla.cg(A, b, x0=x0, rtol=1e-10, atol=0, M=Minv, callback=cb, maxiter=100000)
    print(f"{label:30s} its {it[0]}")
d = A.diagonal()
run(sp.diags(1/d), "point Jacobi")
for G in [148, 74, 37]:
    bounds = np.linspace(0, n, G+1).astype(int)
    blocks = []
    for c in range(G):
        lo, hi = 2*bounds[c], 2*bounds[c+1]
        blk = A[lo:hi, lo:hi].toarray()
        blocks.append(np.linalg.inv(blk))
    M = sp.block_diag(blocks).tocsr()
    run(M, f"block Jacobi exact, {G} blocks")
    # Neumann degree 1 on blocks: M = D^-1 + D^-1 (D - A_blk) D^-1
    Ab = sp.block_diag([A[2*bounds[c]:2*bounds[c+1], 2*bounds[c]:2*bounds[c+1]] for c in range(G)]).tocsr()
    Di = sp.diags(1/d)
    Mn = Di + Di @ (sp.diags(d) - Ab) @ Di
    run(Mn, f"block Neumann-1, {G} blocks")
print("---")
G = 148
bounds = np.linspace(0, n, G+1).astype(int)
Ab = sp.block_diag([A[2*bounds[c]:2*bounds[c+1], 2*bounds[c]:2*bounds[c+1]] for c in range(G)]).tocsr()
Di = sp.diags(1/d); Ds = sp.diags(1/np.sqrt(d))
Ahat = Ds @ Ab @ Ds
lmax = spla.eigsh(Ahat, k=1, which='LA', return_eigenvectors=False)[0]
lmin = spla.eigsh(Ahat, k=1, sigma=0, which='LM', return_eigenvectors=False)[0]
print("block Ahat eig range", lmin, lmax)
E = sp.eye(2*n) - Ab @ Di
M2 = Di @ (sp.eye(2*n) + E + E @ E)
run(sp.csr_matrix(M2), "block Neumann-2, 148 blocks")
Af = Ds @ A @ Ds
print("full Ahat lmax", spla.eigsh(Af, k=1, which='LA', return_eigenvectors=False)[0])
