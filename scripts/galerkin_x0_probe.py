"""CPU study (scipy): total block-Jacobi PCG iterations over the 900 s
mesh-B run for three solver starts: the reference predictor, the device
loops' start (V extrapolated on a step's first pass), and that start
improved by a Galerkin projection onto the last k solution increments
(x0 += W c, (W^T A W) c = W^T r0 with the pass's own A)."""
import sys
import numpy as np
import scipy.sparse as sp
sys.path.insert(0, ".")
from oracle import rafem_oracle as O

dims = (20, 20, 21) if len(sys.argv) < 4 else tuple(int(a) for a in sys.argv[1:4])
mesh = O.box_mesh(*dims)
N = mesh.node_count
geom = O.geometry(mesh)
mats = {0: O.OMaterial()}
G = 148
bounds = [2 * (N * g // G) for g in range(G + 1)]


def bj(A):
    Mi = 1 / A.diagonal()
    blocks = [(lo, hi, A[lo:hi, lo:hi].tocsr()) for lo, hi in zip(bounds[:-1], bounds[1:])]

    def apply(w):
        y = Mi * w
        out = np.empty_like(w)
        for lo, hi, Ab in blocks:
            out[lo:hi] = y[lo:hi] + Mi[lo:hi] * (w[lo:hi] - Ab @ y[lo:hi])
        return out
    return apply


def pcg(A, b, x0, P, tol=1e-10):
    x = x0.copy(); r = b - A @ x; bn = np.linalg.norm(b); its = 0
    while np.linalg.norm(r) / bn > tol:
        z = P(r); p = z.copy(); rz = r @ z
        while True:
            q = A @ p; a = rz / (p @ q); x += a * p; r -= a * q; its += 1
            if np.linalg.norm(r) / bn <= tol:
                break
            z = P(r); rzn = r @ z; p = z + (rzn / rz) * p; rz = rzn
        r = b - A @ x
    return x, its


def run(mode, k=6):
    cfg = O.OSim(total_time=900.0)
    T = np.full(N, cfg.initial_temp); V = np.zeros(N); T_prev = T.copy()
    t, dt_cur, dt_prev, step, passes, inner = 0.0, cfg.dt_init, cfg.dt_init, 0, 0, 0
    hist = []  # previous solutions (for increments)
    ring = []  # mode 3: (correction, A correction) of the last k solves
    ads = []   # modes 5/6: A d_j as computed when d_j was formed
    while t < cfg.total_time:
        remaining = cfg.total_time - t
        last = dt_cur >= remaining
        dt = remaining if last else dt_cur
        t_it = T + (dt / dt_prev) * (T - T_prev) if step >= 1 else T.copy()
        v_it = V.copy()
        x_old = np.empty(2 * N); x_old[0::2], x_old[1::2] = v_it, t_it
        ok, used = False, 0
        for it in range(1, cfg.max_corrector_iters + 1):
            used = it; passes += 1
            s = O.assemble(mesh, mats, cfg.applied_voltage, cfg.boundary_temp, t_it, v_it, T, dt, geom=geom)
            A = sp.csr_matrix((s.vals, s.col_idx, s.row_ptr), shape=(2 * N, 2 * N)); b = s.rhs
            x0 = x_old.copy()
            if mode >= 1 and it == 1 and step >= 1:
                x0[0::2] = V + (dt / dt_prev) * (V - Vp)
            if mode == 3 and len(ring) >= 1:
                # device-friendly: ring of the last k solve corrections d = x_new - x0
                # and their products A d = r0 - r_final (exact with THAT pass's A,
                # stale now); symmetrised Galerkin system, regularised solve
                D = np.stack([d for d, _ in ring], 1); AD = np.stack([ad for _, ad in ring], 1)
                r0 = b - A @ x0
                Mg = D.T @ AD; Mg = 0.5 * (Mg + Mg.T); g = D.T @ r0
                w, U = np.linalg.eigh(Mg)
                keep = w > 1e-12 * w.max()
                c = U[:, keep] @ ((U[:, keep].T @ g) / w[keep])
                x0 = x0 + D @ c
            if mode == 4 and len(hist) >= 2:
                # device form: raw increments, M = D^T A D (current A), scaled
                # Cholesky with a pivot threshold (dependent directions dropped)
                D = np.stack([hist[j] - hist[j - 1] for j in range(max(1, len(hist) - k), len(hist))], 1)
                r0 = b - A @ x0
                AD = A @ D
                Mg = D.T @ AD; g = D.T @ r0
                sc = 1.0 / np.sqrt(np.diag(Mg))
                Ms = Mg * sc[:, None] * sc[None, :]
                kk = Ms.shape[0]; L = np.zeros((kk, kk)); act = np.zeros(kk, bool)
                for i in range(kk):
                    dval = Ms[i, i] - sum(L[i, j] ** 2 for j in range(i) if act[j])
                    if dval > 1e-10:
                        act[i] = True; L[i, i] = np.sqrt(dval)
                        for r_ in range(i + 1, kk):
                            L[r_, i] = (Ms[r_, i] - sum(L[r_, j] * L[i, j] for j in range(i) if act[j])) / L[i, i]
                idx = np.nonzero(act)[0]
                Lr = L[np.ix_(idx, idx)]
                y = np.linalg.solve(Lr, (g * sc)[idx]); cs = np.linalg.solve(Lr.T, y)
                c = np.zeros(kk); c[idx] = cs * sc[idx]
                x0 = x0 + D @ c
            if mode in (5, 6) and len(hist) >= 2:
                # stale products: A d_j from the pass that produced d_j (mode 5),
                # refreshed with the current A on a step's first pass (mode 6)
                D = np.stack([hist[j] - hist[j - 1] for j in range(max(1, len(hist) - k), len(hist))], 1)
                if mode == 6 and it == 1:
                    ads[:] = [None] * len(ads)
                AD = np.stack([ads[j] if ads[j] is not None else A @ (hist[j] - hist[j - 1])
                               for j in range(max(1, len(hist) - k), len(hist))], 1)
                for jj, j in enumerate(range(max(1, len(hist) - k), len(hist))):
                    ads[j] = AD[:, jj]
                r0 = b - A @ x0
                Mg = D.T @ AD; Mg = 0.5 * (Mg + Mg.T); g = D.T @ r0
                w, U = np.linalg.eigh(Mg); keep = w > 1e-12 * w.max()
                c = U[:, keep] @ ((U[:, keep].T @ g) / w[keep])
                x0 = x0 + D @ c
            if mode == 2 and len(hist) >= 2:
                W = np.stack([hist[j] - hist[j - 1] for j in range(max(1, len(hist) - k), len(hist))], 1)
                Q, _ = np.linalg.qr(W)
                AQ = A @ Q
                r0 = b - A @ x0
                c = np.linalg.solve(Q.T @ AQ, Q.T @ r0)
                x0 = x0 + Q @ c
            r0x = b - A @ x0
            x_new, its = pcg(A, b, x0, bj(A))
            inner += its
            if mode == 3:
                ring.append((x_new - x0, r0x - (b - A @ x_new)))
                if len(ring) > k:
                    ring.pop(0)
            hist.append(x_new.copy())
            ads.append(None)
            if len(hist) > k + 1:
                hist.pop(0)
                ads.pop(0)
            delta = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old))))
            v_it, t_it = x_new[0::2].copy(), x_new[1::2].copy(); x_old = x_new
            if delta < cfg.corrector_tol:
                ok = True; break
        assert ok
        Vp = V
        T_prev, T, V = T, t_it, v_it
        dt_prev = dt; t = cfg.total_time if last else t + dt; step += 1
        dt_cur = min(dt * 1.5, cfg.dt_max) if used <= 5 else (max(dt * 0.75, cfg.dt_min) if used >= 20 else dt)
    return step, passes, inner


Vp = None
ks = [int(a) for a in sys.argv[4].split(",")] if len(sys.argv) > 4 else [6]
print("device start (V extrapolated)", run(1), flush=True)
for k in ks:
    print(f"device start + Galerkin k={k} (solution increments, exact A)", run(2, k), flush=True)
    print(f"device start + Galerkin k={k} (raw increments, thresholded Cholesky)", run(4, k), flush=True)
    print(f"device start + Galerkin k={k} (stale A d_j)", run(5, k), flush=True)
    print(f"device start + Galerkin k={k} (A d_j refreshed per step)", run(6, k), flush=True)
