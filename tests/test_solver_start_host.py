"""CPU check of the native loops' first-pass solver start:
starting a step's first PCG solve from V extrapolated in time, while the
pass still assembles from and measures its delta against the reference
predictor, leaves the reference trajectory unchanged.  Runs the oracle's
restatement of run_simulation (fem.py:554-644) with the oracle's PCG."""

import numpy as np

from oracle import rafem_oracle as O


def _run(mesh, cfg, vx0):
    N = mesh.node_count
    geom = O.geometry(mesh)
    mats = {0: O.OMaterial()}
    T = np.full(N, cfg.initial_temp)
    V = np.zeros(N)
    T_prev, V_prev = T.copy(), V.copy()
    t, dt_cur, dt_prev, step = 0.0, cfg.dt_init, cfg.dt_init, 0
    traj, its, fields = [], 0, []
    while t < cfg.total_time:
        remaining = cfg.total_time - t
        last = dt_cur >= remaining
        dt = remaining if last else dt_cur
        t_it = T + (dt / dt_prev) * (T - T_prev) if step >= 1 else T.copy()  # fem.py:445-449
        v_it = V.copy()
        x_old = np.empty(2 * N)
        x_old[0::2], x_old[1::2] = v_it, t_it
        used, ok = 0, False
        for it in range(1, cfg.max_corrector_iters + 1):
            used = it
            s = O.assemble(mesh, mats, cfg.applied_voltage, cfg.boundary_temp, t_it, v_it, T, dt, geom=geom)
            x0 = x_old.copy()
            if vx0 and it == 1 and step >= 1:
                x0[0::2] = V + (dt / dt_prev) * (V - V_prev)
            x_new, st = O.pcg(s.row_ptr, s.col_idx, s.vals, s.rhs.copy(), x0=x0, tol=cfg.tolerance,
                              precondition="jacobi")
            assert st.converged
            its += st.iterations
            delta = float(np.max(np.abs(x_new - x_old) / np.maximum(1.0, np.abs(x_old))))
            v_it, t_it = x_new[0::2].copy(), x_new[1::2].copy()
            x_old = x_new
            if delta < cfg.corrector_tol:
                ok = True
                break
        assert ok
        T_prev, T, V_prev, V = T, t_it, V, v_it
        dt_prev = dt
        t = cfg.total_time if last else t + dt
        traj.append((t, dt, used))
        fields.append((T.copy(), V.copy()))
        step += 1
        dt_cur = min(dt * 1.5, cfg.dt_max) if used <= 5 else (max(dt * 0.75, cfg.dt_min) if used >= 20 else dt)
    return traj, its, fields


def test_v_extrapolated_first_solve_keeps_the_reference_trajectory():
    mesh = O.box_mesh(7, 6, 8)
    cfg = O.OSim(total_time=60.0, method="pcg", tolerance=1e-12)
    ref_traj, ref_its, ref_f = _run(mesh, cfg, vx0=False)
    traj, its, f = _run(mesh, cfg, vx0=True)
    assert traj == ref_traj
    assert its < ref_its
    for (ta, va), (tb, vb) in zip(f, ref_f):
        assert np.max(np.abs(ta - tb)) <= 1e-8 * np.max(np.abs(tb))
        assert np.max(np.abs(va - vb)) <= 1e-8 * max(np.max(np.abs(vb)), 1.0)
