"""CPU study (oracle, analysis only): PCG iterations of the whole 900 s
mesh-B run when corrector pass k >= 2 starts its solve from an
extrapolation of the Picard iterates, x0 = x_k + c (x_k - x_{k-1}),
instead of x_k (the reference passes the current iterate, fem.py:497-501).
The trajectory (accepted steps, passes) must not change.

    python scripts/x0_extrap_probe.py [c ...] [--vfirst]
    (default: the reference x0 vs the first pass's V extrapolated in time)
"""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from oracle import rafem_oracle as O


def run(mesh, cfg, c, precondition="jacobi", vfirst=False, quad=False):
    N = mesh.node_count
    geom = O.geometry(mesh)
    mats = {0: O.OMaterial()}
    T = np.full(N, cfg.initial_temp); V = np.zeros(N); T_prev = T.copy(); V_prev = V.copy()
    T_prev2, V_prev2, dt_prev2 = T.copy(), V.copy(), cfg.dt_init
    first_its = later_its = 0
    t, dt_cur, dt_prev, step = 0.0, cfg.dt_init, cfg.dt_init, 0
    passes = inner = 0
    traj = []
    while t < cfg.total_time:
        remaining = cfg.total_time - t
        last = dt_cur >= remaining
        dt = remaining if last else dt_cur
        t_it = T + (dt / dt_prev) * (T - T_prev) if step >= 1 else T.copy()
        v_it = V.copy()
        x_old = np.empty(2 * N); x_old[0::2], x_old[1::2] = v_it, t_it
        x_prev = None
        ok, used = False, 0
        for it in range(1, cfg.max_corrector_iters + 1):
            used = it
            passes += 1
            s = O.assemble(mesh, mats, cfg.applied_voltage, cfg.boundary_temp, t_it, v_it, T, dt, geom=geom)
            x0 = x_old if (x_prev is None or c == 0.0) else x_old + c * (x_old - x_prev)
            if vfirst and x_prev is None and step >= 1:  # first pass: V extrapolated in time like T
                x0 = x_old.copy()
                x0[0::2] = V + (dt / dt_prev) * (V - V_prev)
                if quad and step >= 2:  # quadratic (Lagrange through the last three accepted steps)
                    t0_, t1_, t2_, te = -dt_prev - dt_prev2, -dt_prev, 0.0, dt
                    l0 = (te - t1_) * (te - t2_) / ((t0_ - t1_) * (t0_ - t2_))
                    l1 = (te - t0_) * (te - t2_) / ((t1_ - t0_) * (t1_ - t2_))
                    l2 = (te - t0_) * (te - t1_) / ((t2_ - t0_) * (t2_ - t1_))
                    x0[0::2] = l0 * V_prev2 + l1 * V_prev + l2 * V
                    x0[1::2] = l0 * T_prev2 + l1 * T_prev + l2 * T
            x_new, st = O.pcg(s.row_ptr, s.col_idx, s.vals, s.rhs.copy(), x0=x0.copy(), tol=cfg.tolerance,
                              precondition=precondition)
            inner += st.iterations
            if x_prev is None:
                first_its += st.iterations
            else:
                later_its += st.iterations
            delta = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old))))
            v_it, t_it = x_new[0::2].copy(), x_new[1::2].copy()
            x_prev, x_old = x_old, x_new
            if delta < cfg.corrector_tol:
                ok = True
                break
        assert ok
        T_prev2, V_prev2, dt_prev2 = T_prev, V_prev, dt_prev
        T_prev, T, V_prev, V = T, t_it, V, v_it
        dt_prev = dt
        t = cfg.total_time if last else t + dt
        traj.append((round(t, 9), used))
        step += 1
        dt_cur = min(dt * 1.5, cfg.dt_max) if used <= 5 else (max(dt * 0.75, cfg.dt_min) if used >= 20 else dt)
    print(f"   first-pass solves {first_its} its, later passes {later_its} its", flush=True)
    return step, passes, inner, traj


mesh = O.box_mesh(20, 20, 21)
cfg = O.OSim(total_time=900.0, method="pcg")
variants = [(0.0, False, False), (0.0, True, False)] if len(sys.argv) == 1 else \
    [(float(a), "--vfirst" in sys.argv, "--quad" in sys.argv) for a in sys.argv[1:] if not a.startswith("--")]
base = None
for c, vfirst, quad in variants:
    t0 = time.perf_counter()
    steps, passes, inner, traj = run(mesh, cfg, c, vfirst=vfirst, quad=quad)
    same = "" if base is None else ("same trajectory" if traj == base else "TRAJECTORY DIFFERS")
    base = base or traj
    print(f"c={c:4.2f} vfirst={vfirst} quad={quad}: steps {steps} passes {passes} PCG iterations {inner} "
          f"({time.perf_counter() - t0:.0f} s) {same}", flush=True)
