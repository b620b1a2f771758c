"""CPU study (scipy): combined-scalar PCG vs split V/T scalars (an alpha/beta
per field) on the mesh-B / mesh-A systems, Jacobi and 148-block block-Jacobi."""
import numpy as np, sys, scipy.sparse as sp
sys.path.insert(0,'.')
from oracle import rafem_oracle as O
from paper_2409_13036_b200 import generate_box_mesh
for dims in [(20,20,21),(15,15,16)]:
    mesh=O.box_mesh(*dims); n=mesh.nodes.shape[0] if hasattr(mesh,'nodes') else None
    m2 = generate_box_mesh(*dims); n=m2.node_count
    rng=np.random.default_rng(2409)
    t=37+rng.uniform(0,30,n); v=rng.uniform(0,25,n)
    r=O.assemble(mesh,{0:O.OMaterial()},25.0,37.0,t,v,t,0.5)
    A=sp.csr_matrix((r.vals,r.col_idx,r.row_ptr),shape=(2*n,2*n)); b=r.rhs
    x0=np.empty(2*n); x0[0::2]=v; x0[1::2]=t
    d=A.diagonal(); Mi=1/d
    def pcg(split, tol=1e-10, maxit=5000):
        x=x0.copy(); rr=b-A@x; z=Mi*rr; p=z.copy()
        mask=[np.arange(2*n)%2==0, np.arange(2*n)%2==1] if split else [np.ones(2*n,bool)]
        rz=[rr[m]@z[m] for m in mask]; bn=np.linalg.norm(b)
        for it in range(1,maxit):
            q=A@p
            for k,m in enumerate(mask):
                pq=p[m]@q[m]
                if pq<=0: continue
                a=rz[k]/pq; x[m]+=a*p[m]; rr[m]-=a*q[m]
            if np.linalg.norm(rr)/bn<=tol: return it, np.linalg.norm(b-A@x)/bn
            z=Mi*rr
            for k,m in enumerate(mask):
                rzn=rr[m]@z[m]; beta=rzn/rz[k] if rz[k]>0 else 0; p[m]=z[m]+beta*p[m]; rz[k]=rzn
        return maxit, None
    print(dims, "combined", pcg(False), "split scalars", pcg(True))

# block-Jacobi (one Neumann step on G contiguous row blocks of nodes)
def bj_apply_factory(A, Mi, G, n):
    N = n
    bounds = [2 * (N * g // G) for g in range(G + 1)]
    blocks = []
    for g in range(G):
        lo, hi = bounds[g], bounds[g + 1]
        blocks.append((lo, hi, A[lo:hi, lo:hi].tocsr()))
    def apply(w):
        y = Mi * w
        out = np.empty_like(w)
        for lo, hi, Ab in blocks:
            out[lo:hi] = y[lo:hi] + Mi[lo:hi] * (w[lo:hi] - Ab @ y[lo:hi])
        return out
    return apply
for dims in [(20,20,21),(15,15,16)]:
    mesh=O.box_mesh(*dims); m2 = generate_box_mesh(*dims); n=m2.node_count
    rng=np.random.default_rng(2409)
    t=37+rng.uniform(0,30,n); v=rng.uniform(0,25,n)
    r=O.assemble(mesh,{0:O.OMaterial()},25.0,37.0,t,v,t,0.5)
    A=sp.csr_matrix((r.vals,r.col_idx,r.row_ptr),shape=(2*n,2*n)); b=r.rhs
    x0=np.empty(2*n); x0[0::2]=v; x0[1::2]=t
    Mi=1/A.diagonal()
    P = bj_apply_factory(A, Mi, 148, n)
    def pcg(split, tol=1e-10, maxit=5000):
        x=x0.copy(); rr=b-A@x; z=P(rr); p=z.copy()
        mask=[np.arange(2*n)%2==0, np.arange(2*n)%2==1] if split else [np.ones(2*n,bool)]
        rz=[rr[m]@z[m] for m in mask]; bn=np.linalg.norm(b)
        for it in range(1,maxit):
            q=A@p
            for k,m in enumerate(mask):
                pq=p[m]@q[m]
                if pq<=0: continue
                a=rz[k]/pq; x[m]+=a*p[m]; rr[m]-=a*q[m]
            if np.linalg.norm(rr)/bn<=tol: return it
            z=P(rr)
            for k,m in enumerate(mask):
                rzn=rr[m]@z[m]; beta=rzn/rz[k] if rz[k]>0 else 0; p[m]=z[m]+beta*p[m]; rz[k]=rzn
        return maxit
    print(dims, "BJ148 combined", pcg(False), "split", pcg(True))
