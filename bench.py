"""Benchmark of the RAFEM hot path on B200.

Metric (BASELINE.json): accepted RAFEM time steps per second of a full
simulation.  Workload (configs[1], "the paper's larger workload"): the
mesh-B analog generate_box_mesh(20, 20, 21) (8,400 nodes, 43,320 tets,
16,800 dofs), the full 900 s simulated ablation (96 accepted steps, 214
corrector passes), GMRES/PCG with Jacobi at tol 1e-10.

One bench step = one full 900 s simulation.
  value : native device loop (rafem_simulate), mesh and state in HBM.
  e2e   : the reference-shaped public API (run_simulation -> assemble_global
          -> solve) with host numpy buffers crossing the boundary every pass.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference algorithm's CPU restatement
(oracle/rafem_oracle.py, a bit-exact numpy port of rafem 0.1.0, pinned
against the reference's golden vectors) on the host cores; each of its
steps is a window of 8 accepted steps of one continuing simulation.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MESH_B = (20, 20, 21)
TOTAL_TIME = 900.0
METRIC = "time-steps/s (full 900 s RAFEM simulation, mesh-B analog)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--backend", default="pcg", choices=["pcg", "gmres"])
    ap.add_argument("--precond", default="block_jacobi", choices=["jacobi", "block_jacobi"],
                    help="PCG preconditioner (GMRES always uses the reference's point Jacobi)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--ref-worker", default=None, help=argparse.SUPPRESS)
    return ap.parse_args()


def prec_of(args):
    """PCG: block-Jacobi (north_star's "Jacobi or block-Jacobi"); GMRES: the
    reference's point Jacobi."""
    return args.precond if args.backend == "pcg" else "jacobi"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


# RAFEM_BENCH_BACKEND=gloo (testing only): ranks may share a GPU and the
# sharded leg stages its collectives through host memory; the job's numbers
# are then not a multi-GPU measurement.
BACKEND = os.environ.get("RAFEM_BENCH_BACKEND", "nccl")


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            self.nv = None
            self.err = str(exc)

    _NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
              0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle",
              0x2: "applications_clocks_setting", 0x100: "display_clock_setting"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU legs (the reference on the host cores; never the measured product)
#
# The reference package (rafem 0.1.0, pure Python + numpy) is staged
# unmodified into baseline/_ref by scripts/stage_reference.sh and driven
# through its own public API (rafem.fem.run_simulation).  Where it is not
# staged, the bit-exact numpy port oracle/rafem_oracle.py stands in
# (kind "port"); the port is ~25 % faster than the reference itself.

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def workload_config():
    """The workload both arms time; identical in both JSON lines."""
    return {"workload": "rafem-B900", "mesh": "generate_box_mesh(20,20,21)", "nodes": 8400, "dofs": 16800,
            "total_time_s": TOTAL_TIME, "accepted_steps_per_run": 96,
            "physics": "MaterialParams.default(), SimConfig() defaults (25 V electrode, 37 C boundary)",
            "tolerance": 1e-10,
            "timed_region": "complete 900 s simulations only: value = accepted steps / wall of whole runs",
            "l2": "GPU arm: flushed (256 MB write) between timed steps"}


def ref_worker(spec: dict) -> dict:
    """One CPU setting of the reference in THIS process (BLAS threads were
    fixed by the parent through the environment before numpy loaded).

    Warm-up: ``warm_steps`` accepted steps of a separate run.  Timed: one
    run from t = 0 with a perf_counter stamp at every accepted step (the
    reference's sink, fem.py:609-610), stopped after ``max_steps`` when
    given, else complete."""
    dims, total = tuple(spec["dims"]), float(spec["total"])
    warm, max_steps, threads = int(spec["warm_steps"]), spec.get("max_steps"), int(spec["threads"])

    class _Stop(Exception):
        pass

    kind = "port"
    if os.path.isdir(os.path.join(REF_DIR, "rafem")):
        sys.path.insert(0, REF_DIR)
        import rafem
        import rafem.fem as F
        from rafem.mesh import generate_box_mesh
        from rafem.solver import SolverConfig
        assert os.path.realpath(rafem.__file__).startswith(os.path.realpath(REF_DIR))
        kind = "reference"
        mesh = generate_box_mesh(*dims)
        mat = F.MaterialParams.default()

        def go(limit, stamps):
            cfg = F.SimConfig(total_time=total, threads=threads,
                              solver=SolverConfig(backend="gmres", precondition="jacobi", tolerance=1e-10))

            def sink(_rec):
                stamps.append(time.perf_counter())
                if limit is not None and len(stamps) >= limit:
                    raise _Stop
            try:
                s = F.run_simulation(mesh, mat, cfg, sink=sink)
                return s.total_corrector_iters, s.total_solver_iterations
            except _Stop:
                return None, None
    else:
        from oracle import rafem_oracle as O
        mesh = O.box_mesh(*dims)

        def go(limit, stamps):
            r = O.run(mesh, {0: O.OMaterial()}, O.OSim(total_time=total), keep_fields=False, max_steps=limit,
                      on_step=lambda _r: stamps.append(time.perf_counter()))
            return r.corrector_passes, r.solver_iterations

    if warm > 0:
        go(warm, [])
    stamps = []
    t0 = time.perf_counter()
    passes, iters = go(max_steps, stamps)
    t1 = time.perf_counter()
    return {"kind": kind, "wall_s": t1 - t0, "stamps": [x - t0 for x in stamps], "steps": len(stamps),
            "passes": passes, "iterations": iters, "threads": threads}


def cpu_run(dims, total, threads: int, warm_steps: int = 0, max_steps=None, timeout=1800) -> dict:
    """ref_worker in a subprocess: 1 thread pins BLAS and the assembly pool
    to one core; threads > 1 leaves BLAS at its default and gives the
    reference's assembly pool (SimConfig.threads, fem.py:368-379) that many."""
    spec = {"dims": list(dims), "total": total, "threads": threads, "warm_steps": warm_steps,
            "max_steps": max_steps}
    env = dict(os.environ)
    if threads == 1:
        env.update(OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-worker", json.dumps(spec)],
                         capture_output=True, text=True, env=env, timeout=timeout)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-2000:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(args):
    """--impl reference: the reference's own CPU path, rafem.fem.run_simulation
    (GMRES(30) + Jacobi at 1e-10, its default iterative configuration), on
    this host's cores.  The timed region is ONE complete 900 s simulation,
    the same unit of work as our arm's step; bench step k is the contiguous
    window of accepted steps [round(96k/K), round(96(k+1)/K)) of that run,
    so the K windows together are exactly the whole run.  Warm-up: W
    windows' worth of accepted steps of a separate run.  Both BASELINE.md
    §2 settings (1 thread; all cores) are timed on that same sample and
    the faster is reported."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    K, W = max(1, args.steps), max(0, args.warmup)
    warm = W * max(1, round(96 / K))
    runs = {}
    for thr in (1, cores):
        runs[thr] = cpu_run(MESH_B, TOTAL_TIME, thr, warm_steps=warm)
    best_thr = max(runs, key=lambda t: runs[t]["steps"] / runs[t]["wall_s"])
    r = runs[best_thr]
    steps, total = r["steps"], r["wall_s"]
    bounds = [round(steps * k / K) for k in range(K + 1)]
    st = [0.0] + r["stamps"]
    windows = [(st[bounds[k + 1]] if k + 1 < K else total) - st[bounds[k]] for k in range(K)]
    value = steps / total
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": args.gpus,
        "steps": K, "warmup": W, "ms_per_step": 1e3 * total / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn box mesh; reference physics defaults)",
        "impl": "reference",
        "config": workload_config(),
        "run": {"solver": "gmres(30)+jacobi tol 1e-10 (the reference's own solver)",
                "path": ("rafem.fem.run_simulation from baseline/_ref (unmodified rafem 0.1.0)"
                         if r["kind"] == "reference" else "oracle/rafem_oracle.py (bit-exact numpy port)"),
                "step": f"window k of ONE complete 900 s run: accepted steps [round({steps}k/{K}), "
                        f"round({steps}(k+1)/{K})); the {K} windows cover the whole run",
                "window_s": windows, "corrector_passes": r["passes"], "solver_iterations": r["iterations"],
                "settings": {f"{t} thread{'s' if t > 1 else ''}": {"wall_s": runs[t]["wall_s"],
                                                                  "steps_per_s": runs[t]["steps"] / runs[t]["wall_s"]}
                             for t in runs},
                "reported": f"{best_thr} thread{'s' if best_thr > 1 else ''} (the faster)"},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": best_thr, "kind": r["kind"],
                         "sample": f"one complete 900 s run ({steps} accepted steps, {r['passes']} passes) after "
                                   f"{warm} warm-up steps; 1 thread and {cores} threads timed, faster reported"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm

def pcg_iter_bytes(N, S):
    """Algorithmic HBM bytes of one fused PCG iteration on the paired layout.

    SpMV: 20 B per slot (int32 column + (V,T) double2) + 4(N+1) row_ptr.
    Vectors, 16 B per node each: SpMV phase reads z, p_old; writes p, q;
    update phase reads x, p, r, q, minv; writes x, r, z  -> 12 x 16N.
    """
    return 20 * S + 4 * (N + 1) + 12 * 16 * N


def asm_pass_bytes(N, S, M):
    """Algorithmic bytes of one device assembly (element + fill + constraints):
    per tet 16 B tets + 13 geometry doubles read (base 10, vol, 2 field
    gathers amortised per node) + 16 (V, T) contributions and 4 loads
    written then read; per slot 20 B written (fill) and read + written
    (constraints); per node rhs / diagonal / minv 48 B."""
    return M * (16 + 8 * 13 + 2 * (16 * 16 + 32)) + S * (20 + 36) + 48 * N


def galerkin_start_bytes(N, S, k):
    """Algorithmic bytes of one Galerkin solver start with a window of k
    increments (simulate_dev.cuh galerkin_start): 1 + k slice products (the
    matrix, the source and the product per product), the k increment rows
    read once, x0 and r0 read and written."""
    return (1 + k) * (20 * S + 4 * (N + 1) + 32 * N) + k * 16 * N + 4 * 16 * N


def gmres_iter_bytes(N, S, k_avg):
    """GMRES(m) CGS2 step k: SpMV + 2 passes over k+1 basis vectors + updates."""
    n = 2 * N
    return 20 * S + 4 * (N + 1) + 16 * N + (32 * (k_avg + 1) + 56) * n


def run_ours(args):
    import torch
    rank, local, world = dist_env()
    if BACKEND != "nccl":
        local = local % max(1, torch.cuda.device_count())
    os.environ["RAFEM_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        import datetime
        # a collective that never completes aborts the job instead of hanging it
        dist.init_process_group(BACKEND, init_method="env://", timeout=datetime.timedelta(seconds=600))
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh, run_simulation
    from paper_2409_13036_b200.timeloop import DeviceRun

    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"

    mesh = generate_box_mesh(*MESH_B)
    mat = MaterialParams.default()
    cfg = SimConfig(total_time=TOTAL_TIME, solver=SolverConfig(backend=args.backend, precondition=prec_of(args)))
    runner = DeviceRun(mesh, mat)
    stream = torch.cuda.ExternalStream(nat.lib().rafem_stream(nat.context()))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2

    def one(record):
        recs, summ = runner.run(cfg, record_fields=record)
        return summ

    for _ in range(args.warmup):
        one(False)
    launches0 = nat.kernel_launches()
    times, summs = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            summs.append(one(False))
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            torch.cuda.synchronize()
    launches = nat.kernel_launches() - launches0
    total_ms = float(sum(times))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    steps_per_run = summs[0].accepted_steps
    value = world * args.steps * steps_per_run / (total_ms / 1e3)

    # roofline of the dominant kernel: simulate_kernel, one cooperative launch
    # per timed step (the whole 900 s run).  Algorithmic bytes per launch:
    # every PCG iteration (SpMV + vector updates) and every corrector pass
    # (assembly fill + constraint pass over the matrix, rhs, iterates).
    S, N, M = runner.dm.slots, runner.dm.node_count, runner.dm.tet_count
    iters = sum(s.total_solver_iterations for s in summs)
    passes = sum(s.passes for s in summs)
    solve_ms = sum(s.solve_ms for s in summs)
    asm_ms = sum(s.assemble_ms for s in summs)
    pass_bytes = (20 * S + 4 * (N + 1) + 6 * 16 * N) + asm_pass_bytes(N, S, M)
    gal_k = int(os.environ.get("RAFEM_GALERKIN_K", "14"))
    gal_starts = 0
    if args.backend == "pcg":
        # the fused simulation starts every pass but a run's first from the
        # Galerkin projection (block-Jacobi PCG)
        if runner.last_mode == "fused-simulation" and prec_of(args) == "block_jacobi" and gal_k > 0:
            gal_starts = passes - len(summs)
        bytes_total = (iters * pcg_iter_bytes(N, S) + passes * pass_bytes
                       + gal_starts * galerkin_start_bytes(N, S, gal_k))
    else:
        bytes_total = iters * gmres_iter_bytes(N, S, 15) + passes * pass_bytes
    fused = runner.last_mode == "fused-simulation"
    launches = args.steps if fused else passes
    launch_ms = total_ms / args.steps if fused else solve_ms / max(passes, 1)
    achieved = bytes_total / launches / (launch_ms / 1e3) / 1e9 if launch_ms > 0 else 0.0
    # DRAM traffic of one launch from the committed ncu --set full capture of
    # the same run (scripts/ncu_summary.py -> profiles/traffic.json)
    traffic = None
    tj = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tj):
        try:
            traffic = json.load(open(tj)).get("simulate_kernel") if fused else None
        except Exception:  # noqa: BLE001
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic,
                "traffic_source": ("DRAM bytes of one launch from the committed ncu --set full capture "
                                   "(profiles/traffic.json), not measured in this run") if traffic else None,
                "kernel": ("simulate_kernel (whole 900 s run in one cooperative launch)" if fused
                           else f"{args.backend}_grid_kernel (persistent solve)"),
                "launches": launches, "avg_launch_us": 1e3 * launch_ms,
                "bytes_per_launch": bytes_total / launches,
                "share_of_step": (launch_ms * launches / total_ms) if world == 1 else None,
                "peak_source": peak_src,
                "galerkin_starts": gal_starts, "galerkin_window": gal_k if gal_starts else 0,
                "bytes_formula": ("PCG iterations x pcg_iter_bytes + passes x (assembly + pass vectors) + "
                                  "Galerkin starts x galerkin_start_bytes (window k; the first passes' "
                                  "windows are shorter, so this slightly overstates)"),
                "note": "paper-scale mesh: the working set (~5 MB) lives in L2 and shared memory, so the "
                        "kernel is bound by grid-barrier + L2 round-trip latency "
                        f"({1e3 * solve_ms / max(iters, 1):.2f} us of solve per PCG iteration, heads included), "
                        "not HBM; the HBM-bound kernels are reported in spmv_c3 and sharded_c4"}

    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generated Kuhn box mesh; reference physics defaults)",
        "config": workload_config(),
        "run": {"slots": S, "accepted_steps_per_run": steps_per_run,
                "corrector_passes_per_run": summs[0].passes,
                "solver_iterations_per_run": summs[0].total_solver_iterations,
                "solver": f"{args.backend}+{prec_of(args)} tol 1e-10", "parallelism": f"replicas x{world}",
                "step": "one complete 900 s simulation",
                "device_path": f"{runner.last_mode} ({runner.last_ctas} CTAs)",
                "assemble_ms_per_run": asm_ms / args.steps, "solve_ms_per_run": solve_ms / args.steps},
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    if not args.no_e2e:  # every rank runs its replica; the legs take the max wall over ranks
        e2e = e2e_leg(mesh, mat, args, SimConfig, SolverConfig, world)
        seam = e2e_plugin_leg(mesh, mat, args, run_simulation, SimConfig, SolverConfig, world)
        # the reference's own solver configuration through the seam: device GMRES(30) + Jacobi
        ga = argparse.Namespace(**vars(args))
        ga.backend, ga.steps = "gmres", 1
        seam_g = e2e_plugin_leg(mesh, mat, ga, run_simulation, SimConfig, SolverConfig, world)
        if rank == 0:
            line["e2e"], line["e2e_plugin_seam"], line["e2e_plugin_seam_gmres"] = e2e, seam, seam_g
    if rank == 0 and not args.no_c3:
        try:
            line["spmv_c3"] = c3_leg(hbm_peak, peak_src, cpu_on=not args.no_cpu)
        except Exception as exc:  # noqa: BLE001
            line["spmv_c3"] = {"error": str(exc)[:300]}
    if rank == 0 and not args.no_c3:
        try:
            line["paper_solve"] = paper_solve_leg()
        except Exception as exc:  # noqa: BLE001
            line["paper_solve"] = {"error": str(exc)[:300]}
    if rank == 0 and not args.no_c3:
        try:
            line["small_c1"] = c1_leg(args)
        except Exception as exc:  # noqa: BLE001
            line["small_c1"] = {"error": str(exc)[:300]}
    if rank == 0 and not args.no_cpu:
        try:
            smp = cpu_run(MESH_B, TOTAL_TIME, 1, warm_steps=2, max_steps=24)
            line["cpu_baseline"] = {"value": smp["steps"] / smp["wall_s"], "unit": "steps/s", "cores": 1,
                                    "kind": smp["kind"],
                                    "sample": f"first {smp['steps']} accepted steps of the same 900 s run "
                                              f"({smp['wall_s']:.1f} s), "
                                              + ("rafem.fem.run_simulation (baseline/_ref)" if smp["kind"] == "reference"
                                                 else "bit-exact numpy port of rafem 0.1.0")
                                              + ", GMRES(30)+Jacobi 1e-10, 1 thread; the --impl reference arm "
                                                "times whole runs at 1 and all threads"}
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"error": str(exc)[:300]}
    # Multi-GPU jobs: the sharded leg is the only one with collectives on the
    # data path.  A watchdog on every rank guarantees the line is printed and
    # the job ends even if a collective never completes.
    import threading
    printed = threading.Event()

    def emit():
        if rank == 0 and not printed.is_set():
            printed.set()
            print(json.dumps(line), flush=True)

    def guard(seconds, what):
        def fire():
            if rank == 0 and what and "sharded_c4" not in line:
                line["sharded_c4"] = {"error": what}
            emit()
            os._exit(0)
        t = threading.Timer(seconds, fire)
        t.daemon = True
        if world > 1:
            t.start()
        return t

    if not args.no_c4:
        wd = guard(480, "sharded leg did not finish within 480 s (watchdog)")
        try:
            c4 = c4_leg(hbm_peak, peak_src, world, rank, local)
        except Exception as exc:  # noqa: BLE001
            c4 = {"error": str(exc)[:300]}
        wd.cancel()
        if rank == 0:
            line["sharded_c4"] = c4
    if not args.no_c5 and world == 1:
        try:
            line["c5_1gpu"] = c5_leg(hbm_peak, peak_src)
        except Exception as exc:  # noqa: BLE001
            line["c5_1gpu"] = {"error": str(exc)[:300]}
    emit()
    if world > 1:
        import torch.distributed as dist
        guard(120, None)  # teardown must not hang the job either
        try:
            dist.barrier()
            dist.destroy_process_group()
        except Exception:  # noqa: BLE001 - the line is already printed
            pass


def _job_wall(wall, world):
    """Max of a wall-clock interval over the job's ranks (NCCL all-reduce)."""
    if world <= 1:
        return wall
    import torch
    import torch.distributed as dist
    t = torch.tensor([wall], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _align(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def e2e_leg(mesh, mat, args, SimConfig, SolverConfig, world):
    """Same metric end to end through the public whole-simulation API
    (simulate_device -> rafem_mesh_create + rafem_simulate): every step
    uploads the host mesh (nodes, tets, regions, Dirichlet kinds) from host
    memory, runs the symbolic phase, and reads every accepted step's V/T
    fields back to host arrays."""
    from paper_2409_13036_b200.timeloop import DeviceRun
    cfg = SimConfig(total_time=TOTAL_TIME, solver=SolverConfig(backend=args.backend, precondition=prec_of(args)))

    def one():
        recs = []
        summ = DeviceRun(mesh, mat, cached=False).run_streamed(cfg, recs.append)
        return recs, summ

    one()  # warm
    reps = max(1, args.steps)
    _align(world)
    t0 = time.perf_counter()
    for _ in range(reps):
        recs, summ = one()
    wall = _job_wall(time.perf_counter() - t0, world)
    N, M = mesh.node_count, mesh.tet_count
    h2d = 8 * 3 * N + 8 * 4 * M + 4 * M + 2 * N + 5 * 8  # nodes f64, tets i64, region idx i32, dof kinds u8, tables
    d2h = len(recs) * (16 * N + 8 + 8 + 8 + 4) + 128  # per accepted step: V/T fields, step/time/dt/iters; summary
    # whole job: every rank runs its own simulation (replicas), slowest rank's wall
    return {"value": world * int(summ.accepted_steps) * reps / wall, "unit": "steps/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "reps": reps,
            "path": "DeviceRun(cached=False).run_streamed: host mesh -> rafem_mesh_create -> "
                    "rafem_simulate_stream -> host fields of every accepted step, streamed while the kernel runs "
                    "(wall clock)"}


def e2e_plugin_leg(mesh, mat, args, run_simulation, SimConfig, SolverConfig, world):
    """Same metric through the reference's plug-in seam: the REFERENCE's own
    rafem.fem.run_simulation (unmodified, staged in baseline/_ref) with
    plugin.install() routing its corrector's assemble_global / solve to the
    device (fem.py:47-48, 492, 501); host numpy buffers cross the boundary
    every corrector pass.  Where the reference is not staged, this
    package's mirror of run_simulation (timeloop.py) stands in and the leg
    says so."""
    ref_ok = os.path.isdir(os.path.join(REF_DIR, "rafem"))
    if ref_ok:
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import rafem.fem as F
        from rafem.mesh import generate_box_mesh as ref_box
        from rafem.solver import SolverConfig as RefSolverConfig
        from paper_2409_13036_b200 import plugin
        solver = "pcg" if args.backend == "pcg" else None
        plugin.install("rafem.fem", solver=solver, precondition=prec_of(args) if solver else None)
        rmesh, rmat = ref_box(*MESH_B), F.MaterialParams.default()
        cfg = F.SimConfig(total_time=TOTAL_TIME, solver=RefSolverConfig(backend="gmres", precondition="jacobi"))

        def go():
            return F.run_simulation(rmesh, rmat, cfg)
        path = ("rafem.fem.run_simulation (reference, baseline/_ref) -> plugin seam -> device assemble_global + "
                + ("device PCG (install(solver='pcg'))" if solver else "device GMRES(30)+Jacobi")
                + "; host numpy in/out every corrector pass")
    else:
        cfg = SimConfig(total_time=TOTAL_TIME, solver=SolverConfig(backend=args.backend, precondition=prec_of(args)))

        def go():
            return run_simulation(mesh, mat, cfg)
        path = "timeloop.run_simulation (this package's mirror; reference not staged) -> assemble_global -> solve"
    try:
        go()  # warm (mesh upload + symbolic phase cached)
        reps = max(1, min(args.steps, 3))
        _align(world)
        t0 = time.perf_counter()
        for _ in range(reps):
            summ = go()
        wall = _job_wall(time.perf_counter() - t0, world)
    finally:
        if ref_ok:
            plugin.uninstall("rafem.fem")
    N = mesh.node_count
    passes = summ.total_corrector_iters
    # per pass: H2D t_iter, v_iter, t_prev (3N f64) + b, x0 (2 x 2N f64); D2H rhs + x (2 x 2N f64)
    h2d = passes * 8 * (3 * N + 4 * N)
    d2h = passes * 8 * (4 * N) + passes * 16
    return {"value": world * summ.accepted_steps * reps / wall, "unit": "steps/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "reps": reps, "reference_driven": ref_ok, "path": path}


def paper_solve_leg():
    """Standalone paper-scale solve (the plug-in seam's solve() path): the
    mesh-B analog's system at a hot iterate (seeded fields), PCG to 1e-10
    from the iterate, on the cluster-resident engine (one 16-CTA cluster,
    DSMEM halos, cluster.cu; the default for paper-scale PCG) and on the
    148-CTA grid engine (RAFEM_CLUSTER=0), best of 5 device-timed solves."""
    import numpy as np
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    from paper_2409_13036_b200 import _native as nat
    mesh = generate_box_mesh(*MESH_B)
    n = mesh.node_count
    rng = np.random.default_rng(2409)
    t = 37 + rng.uniform(0, 30, n)
    v = rng.uniform(0, 25, n)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, v, t, 0.5)
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = v, t
    out = {"workload": "generate_box_mesh(20,20,21) system at a seeded hot iterate, x0 = iterate, tol 1e-10"}
    for prec in ("jacobi", "block_jacobi"):
        for eng in ("cluster", "grid"):
            if eng == "grid":
                os.environ["RAFEM_CLUSTER"] = "0"
            try:
                best, st = 1e9, None
                for _ in range(5):
                    x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="pcg", precondition=prec))
                    best = min(best, st.device_ms * 1e3)
                mode = nat.last_solve_mode()
            finally:
                os.environ.pop("RAFEM_CLUSTER", None)
            out[f"{eng}_{prec}"] = {"iterations": st.iterations, "solve_us": best,
                                    "us_per_iteration": best / max(st.iterations, 1),
                                    "engine": {5: "cluster-resident PCG (16 CTAs)", 0: "grid PCG (148 CTAs)"}.get(
                                        mode[0], str(mode)), "ctas": mode[1]}
    return out


def c1_leg(args):
    """configs[0]: the mesh-A analog (15x15x16, 7,200 dofs), 40 s simulated
    (10 accepted steps), native loop vs the CPU port on one core."""
    import torch
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200.timeloop import DeviceRun
    from paper_2409_13036_b200 import _native as nat
    mesh = generate_box_mesh(15, 15, 16)
    cfg = SimConfig(total_time=40.0, solver=SolverConfig(backend=args.backend, precondition=prec_of(args)))
    run = DeviceRun(mesh, MaterialParams.default())
    for _ in range(3):
        run.run(cfg, record_fields=False)
    stream = torch.cuda.ExternalStream(nat.lib().rafem_stream(nat.context()))
    times = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, summ = run.run(cfg, record_fields=False)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    out = {"workload": "generate_box_mesh(15,15,16), 40 s simulated", "accepted_steps": int(summ.accepted_steps),
           "corrector_passes": int(summ.passes), "ms_per_run": ms,
           "steps_per_s": int(summ.accepted_steps) / (ms / 1e3)}
    if not args.no_cpu:
        try:
            c = cpu_run((15, 15, 16), 40.0, 1, warm_steps=0, timeout=600)
            out["cpu_baseline"] = {"kind": c["kind"], "cores": 1, "wall_s": c["wall_s"],
                                   "steps_per_s": c["steps"] / c["wall_s"],
                                   "sample": "the whole 40 s run, GMRES(30)+Jacobi 1e-10"}
            out["speedup_vs_cpu"] = c["wall_s"] / (ms / 1e3)
        except Exception as exc:  # noqa: BLE001
            out["cpu_baseline"] = {"error": str(exc)[:300]}
    return out


def c4_leg(hbm_peak, peak_src, world, rank, local):
    """configs[3]: 16M-dof box, row-block sharded over the job's GPUs (one
    shard per rank, NCCL halo exchange + scalar all-gathers between the
    kernel-per-phase PCG phases); a cold solve to 1e-10."""
    import torch
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, generate_box_mesh
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200.shard import ShardComm, ShardedSystem
    t0 = time.perf_counter()
    mesh = generate_box_mesh(200, 200, 200)
    n = mesh.node_count
    comm = None
    if world > 1:
        stream = torch.cuda.ExternalStream(nat.lib().rafem_stream(nat.context()))
        comm = ShardComm(device_collectives=BACKEND == "nccl", stream=stream)
    sh = ShardedSystem(mesh, MaterialParams.default(), comm, batch=16)
    p = sh.plan
    tt = np.full(n, 37.0)
    t_ext, v_ext = p.extend(tt), np.zeros(p.n_ext)
    sh.assemble(t_ext, v_ext, t_ext, 0.5, SimConfig())  # warm
    setup_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    a0 = time.perf_counter()
    sh.assemble(t_ext, v_ext, t_ext, 0.5, SimConfig())
    asm_s = time.perf_counter() - a0
    x0 = np.empty(2 * p.n_own)
    x0[0::2], x0[1::2] = 0.0, 37.0
    cfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10)
    sh.solve(x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10,
                                        max_total_iters=20))  # warm (communicators, caches)
    x, st = sh.solve(x0=x0, config=cfg)
    dev_ms, wall_ms = float(st.device_ms), st.wall_ns / 1e6
    own_slots = int(sh.dm.dof_row_ptr[2 * p.n_own] // 2)
    cls_on = (int(nat.lib().rafem_mesh_stencil_classes(sh.dm.handle)) > 0
              and os.environ.get("RAFEM_NO_CLASSES", "0") != "1")
    # KP iteration bytes of this shard: SpMV (20 B/slot, or 16 B/slot + 1 B/row
    # with stencil-class columns) + 7 vector reads / 5 writes + u gather + w write
    mine = ((16 * own_slots + p.n_own) if cls_on else 20 * own_slots) + 4 * (p.n_own + 1) + 14 * 16 * p.n_own
    if world > 1:
        import torch.distributed as dist
        tt_ = torch.tensor([dev_ms, wall_ms, asm_s], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        dev_ms, wall_ms, asm_s = (float(v) for v in tt_.tolist())
        s_ = torch.tensor([float(mine)], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(s_)
        mine = int(s_.item())
    it = st.iterations
    bytes_it = mine
    spmv = None
    if world == 1:  # the standalone SpMV on the same matrix, cold L2 every launch
        import ctypes as C
        msb = C.c_double()
        nat.check(nat.lib().rafem_system_spmv_bench(sh.h.handle, 10, 1, C.byref(msb)), "spmv bench")
        S1 = sh.dm.slots
        b_sp = ((16 * S1 + n) if cls_on else 20 * S1) + 4 * (n + 1) + 32 * n
        b_ex = 20 * S1 + 4 * (n + 1) + 32 * n
        ach_sp = b_sp / (msb.value / 1e3) / 1e9
        spmv = {"bound": "hbm", "achieved": ach_sp, "peak": hbm_peak, "unit": "GB/s", "frac": ach_sp / hbm_peak,
                "frac_of_8TBs": ach_sp / 8000.0, "us_per_launch": 1e3 * msb.value, "bytes_per_launch": b_sp,
                "kernel": "spmv_tma_pipe_kernel<192,2,stencil classes>" if cls_on else "spmv_tma_pipe_kernel<256,2>",
                "l2": "flushed (256 MB write) before every timed launch"}
        # the general-mesh layout (explicit int32 columns, 20 B per slot),
        # measured on the same matrix: what an unstructured mesh streams
        try:
            spmv["explicit_columns"] = explicit_leg(sh, n, S1, b_ex, hbm_peak, x0, it)
        except Exception as exc:  # noqa: BLE001
            spmv["explicit_columns"] = {"error": str(exc)[:200]}
    ach = it * bytes_it / (dev_ms / 1e3) / 1e9 if dev_ms > 0 else 0.0
    # configs[3]'s run itself: 10 accepted steps (total_time 40 s), every
    # corrector pass re-assembled, fields resident in HBM on every shard
    loop = None
    try:
        loop = time_loop_leg(sh, comm, world, local, hbm_peak, peak_src, bytes_it, cls_on)
    except Exception as exc:  # noqa: BLE001
        loop = {"error": str(exc)[:300]}
    return {"workload": "generate_box_mesh(200,200,200) cold system, 16,000,000 dofs",
            "time_loop": loop,
            "shards": world, "partition": "contiguous node-row blocks (x-slabs)",
            "collectives": ("none (one shard)" if world == 1 else
                            "NCCL halo send/recv + per-shard scalar all-gather" if BACKEND == "nccl" else
                            f"host-staged {BACKEND} (test backend, ranks may share a GPU)"),
            "iterations": it, "converged": bool(st.converged), "final_relative_residual": st.final_relative_residual,
            "solve_device_ms_max_over_ranks": dev_ms, "solve_wall_ms": wall_ms,
            "us_per_iteration": 1e3 * dev_ms / max(it, 1),
            "aggregate_GBs": ach, "frac_of_1gpu_peak": ach / hbm_peak / world, "peak_source": peak_src,
            "bytes_per_iteration": bytes_it, "columns": "stencil classes" if cls_on else "explicit int32",
            "assembly_s": asm_s, "setup_s": setup_s, "spmv": spmv,
            "kernel": "kp_spmv_kernel + kp_update_kernel (csrc/shard.cu)"}


def explicit_leg(sh, n, S, b_ex, hbm_peak, x0, it_classes, handle=None):
    """SpMV and cold PCG with explicit int32 columns (RAFEM_NO_CLASSES=1:
    no stencil classes, the layout of a general tetrahedral mesh) on a
    single-shard system, timed like the class layout."""
    import ctypes as C
    from paper_2409_13036_b200 import SolverConfig
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200.shard import KPDeviceEngine, ShardedPCG
    os.environ["RAFEM_NO_CLASSES"] = "1"
    try:
        ms = C.c_double()
        h = handle if handle is not None else sh.h.handle
        nat.check(nat.lib().rafem_system_spmv_bench(h, 10, 1, C.byref(ms)), "spmv bench")
        eng = KPDeviceEngine(h, n, n, 1, 0, None)
        pcg = ShardedPCG(eng, None, None, batch=16)
        from paper_2409_13036_b200.krylov import _params
        cfg = SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10)
        pcg.solve(None, x0, _params(cfg, nat.METHOD_PCG), 1 << 14)
        _, st = pcg.solve(None, x0, _params(cfg, nat.METHOD_PCG), 1 << 14)
        eng.close()
    finally:
        del os.environ["RAFEM_NO_CLASSES"]
    it_bytes = 20 * S + 4 * (n + 1) + 14 * 16 * n
    ach = b_ex / (ms.value / 1e3) / 1e9
    pach = st.iterations * it_bytes / (st.device_ms / 1e3) / 1e9 if st.device_ms > 0 else 0.0
    return {"spmv": {"us_per_launch": 1e3 * ms.value, "bytes_per_launch": b_ex, "achieved": ach,
                     "frac": ach / hbm_peak, "unit": "GB/s", "l2": "flushed before every timed launch",
                     "kernel": "spmv_tma_pipe_kernel<256,2> (explicit columns)"},
            "pcg": {"iterations": st.iterations, "iterations_with_classes": it_classes,
                    "us_per_iteration": 1e3 * st.device_ms / max(st.iterations, 1), "bytes_per_iteration": it_bytes,
                    "achieved": pach, "frac": pach / hbm_peak, "unit": "GB/s",
                    "kernel": "kp_spmv_kernel<explicit> + kp_update_kernel"},
            "measured": "in this run (not rescaled)"}


def time_loop_leg(sh, comm, world, local, hbm_peak, peak_src, bytes_it, cls_on, total=40.0):
    """run_simulation over the shards with the device-resident loop
    (shard.DeviceShardedSimulation): `total` simulated seconds (10 steps of
    the default 4 s), re-assembly every corrector pass."""
    import torch
    from paper_2409_13036_b200 import SimConfig, SolverConfig
    from paper_2409_13036_b200.shard import DeviceShardedSimulation
    cfg = SimConfig(total_time=total, solver=SolverConfig(backend="pcg", precondition="jacobi", tolerance=1e-10))
    loop = DeviceShardedSimulation(sh, comm)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    recs, sm = loop.run(cfg)
    torch.cuda.synchronize()
    wall, asm_s, sol_s, sol_dev = sm.wall_s, sm.assemble_s, sm.solve_s, sm.solve_device_ms
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([wall, asm_s, sol_s, sol_dev], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall, asm_s, sol_s, sol_dev = (float(v) for v in t.tolist())
    loop.close()
    N, S, M = sh.dm.node_count, sh.dm.slots, sh.dm.tet_count
    # assembly roofline: element phase + slot fill + constraints of the shard (asm_pass_bytes)
    asm_bytes = asm_pass_bytes(N, S, M)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(asm_bytes)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t)
        asm_bytes = float(t.item())
    asm_ach = sm.passes * asm_bytes / asm_s / 1e9 if asm_s > 0 else 0.0
    sol_ach = sm.total_solver_iterations * bytes_it / (sol_dev / 1e3) / 1e9 if sol_dev > 0 else 0.0
    return {"total_time_s": total, "accepted_steps": sm.accepted_steps, "corrector_passes": sm.passes,
            "solver_iterations": sm.total_solver_iterations, "wall_s": wall,
            "steps_per_s": sm.accepted_steps / wall if wall > 0 else 0.0,
            "assemble_s": asm_s, "solve_s": sol_s, "solve_device_ms": sol_dev,
            "assemble_ms_per_pass": 1e3 * asm_s / max(sm.passes, 1),
            "us_per_pcg_iteration": 1e3 * sol_dev / max(sm.total_solver_iterations, 1),
            "solve_roofline": {"bound": "hbm", "achieved": sol_ach, "peak": hbm_peak * world, "unit": "GB/s",
                               "frac": sol_ach / hbm_peak / world, "bytes_per_iteration": bytes_it,
                               "peak_source": peak_src},
            "assembly_roofline": {"bound": "hbm", "achieved": asm_ach, "peak": hbm_peak * world, "unit": "GB/s",
                                  "frac": asm_ach / hbm_peak / world, "bytes_per_pass": asm_bytes,
                                  "formula": "bench.asm_pass_bytes (element + fill + constraints, wall clock "
                                             "of the pass incl. the sums' reduction)",
                                  "peak_source": peak_src},
            "fields": "device-resident (rafem_sl_*): per pass a 4-double halo per boundary node, the "
                      "equilibration sums and one corrector-delta scalar cross the host",
            "solver": "kernel-per-phase PCG + Jacobi 1e-10"}


def c5_leg(hbm_peak, peak_src):
    """configs[4] on one GPU: the ~64M-dof box (318^3 nodes, 63.9M dofs)
    built on the device, 10 steps with re-assembly every corrector pass."""
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200.assembly import DeviceMesh
    from paper_2409_13036_b200.shard import ShardedSystem
    t0 = time.perf_counter()
    dm = DeviceMesh.from_box(318, 318, 318)
    sh = ShardedSystem.from_device_mesh(dm, batch=16)
    setup_s = time.perf_counter() - t0
    N, S = dm.node_count, dm.slots
    cls_on = (int(nat.lib().rafem_mesh_stencil_classes(dm.handle)) > 0
              and os.environ.get("RAFEM_NO_CLASSES", "0") != "1")
    bytes_it = ((16 * S + N) if cls_on else 20 * S) + 4 * (N + 1) + 14 * 16 * N
    out = time_loop_leg(sh, None, 1, 0, hbm_peak, peak_src, bytes_it, cls_on)
    out.update({"workload": f"generate_box_mesh(318,318,318) on the device, {2 * N:,} dofs, 10 steps "
                            "(total_time 40 s), re-assembly every corrector pass",
                "shards": 1, "setup_s": setup_s, "columns": "stencil classes" if cls_on else "explicit int32",
                "hbm_gb_in_use": None})
    try:
        import torch
        free, total = torch.cuda.mem_get_info()
        out["hbm_gb_in_use"] = (total - free) / 1e9
    except Exception:  # noqa: BLE001
        pass
    return out


def c3_leg(hbm_peak, peak_src, cpu_on=True):
    """1M-dof roofline study (configs[2]): SpMV and cold PCG solve on the device."""
    from paper_2409_13036_b200 import MaterialParams, SimConfig, SolverConfig, assemble_global, generate_box_mesh, solve
    mesh = generate_box_mesh(80, 80, 79)
    n = mesh.node_count
    t = np.full(n, 37.0)
    s = assemble_global(mesh, MaterialParams.default(), SimConfig(), t, np.zeros(n), t, 0.5)
    h = s.device
    import ctypes as C
    from paper_2409_13036_b200 import _native as nat
    ms = C.c_double()
    nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 50, 1, C.byref(ms)), "spmv bench")
    # SURVEY §8(d) C3 protocol: 1,000 back-to-back SpMVs (no flush; the
    # 137 MB stream exceeds the 126 MB L2, and the matrix is marked
    # evict-first), with and without programmatic dependent launch
    ms_b2b, ms_b2b_plain = C.c_double(), C.c_double()
    nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 1000, 0, C.byref(ms_b2b)), "spmv bench")
    os.environ["RAFEM_NO_PDL"] = "1"
    nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 1000, 0, C.byref(ms_b2b_plain)), "spmv bench")
    del os.environ["RAFEM_NO_PDL"]
    b2b_dram = None  # DRAM bytes of one launch inside a back-to-back chain (committed ncu capture)
    try:
        with open(os.path.join(ROOT, "profiles", "r1k_spmv_c3_back_to_back_ncu.txt")) as fh:
            rows = [ln.split() for ln in fh if ln[:1].isdigit()]
        b2b_dram = sum(int(r[1]) + int(r[2]) for r in rows) / len(rows) if rows else None
    except (OSError, ValueError, IndexError):
        pass
    os.environ["RAFEM_NO_TMA_SPMV"] = "1"
    ms_plain = C.c_double()
    nat.check(nat.lib().rafem_system_spmv_bench(h.handle, 50, 1, C.byref(ms_plain)), "spmv bench")
    del os.environ["RAFEM_NO_TMA_SPMV"]
    S, N = h.mesh.slots, n
    ncls = int(nat.lib().rafem_mesh_stencil_classes(h.mesh.handle))
    cls_on = ncls > 0 and os.environ.get("RAFEM_NO_CLASSES", "0") != "1"
    b_explicit = 20 * S + 4 * (N + 1) + 16 * N + 16 * N
    # bytes of the layout the kernel streams: with stencil classes only the
    # (V, T) values per slot plus a class byte per row
    b_paired = (16 * S + N + 4 * (N + 1) + 32 * N) if cls_on else b_explicit
    b_csr = 12 * (2 * S) + 4 * (2 * N + 1) + 8 * 2 * N + 8 * 2 * N
    ach = b_paired / (ms.value / 1e3) / 1e9
    x0 = np.empty(2 * n)
    x0[0::2], x0[1::2] = 0.0, 37.0
    import torch
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi"))  # warm
    flush.fill_(2.0)
    torch.cuda.synchronize()
    x, st = solve(s.matrix, s.rhs, x0=x0, config=SolverConfig(backend="pcg", precondition="jacobi"))
    del flush
    mode = nat.last_solve_mode()[0]
    try:
        expl = explicit_leg(None, N, S, b_explicit, hbm_peak, x0, st.iterations, handle=h.handle)
    except Exception as exc:  # noqa: BLE001
        expl = {"error": str(exc)[:200]}
    if mode == 4:  # kernel-per-phase engine: its SpMV bytes + 7 vector reads / 5 writes + u gather + w write
        it_bytes = ((16 * S + N) if cls_on else 20 * S) + 4 * (N + 1) + 14 * 16 * N
    else:
        it_bytes = pcg_iter_bytes(N, S)
    solve_ach = st.iterations * it_bytes / (st.device_ms / 1e3) / 1e9 if st.device_ms else 0.0
    cpu = {}
    if cpu_on:
        # the same matrix through the oracle port (reference arithmetic) on 1 core
        try:
            from oracle import rafem_oracle as O
            a = s.matrix
            rp, ci, va = a.row_ptr, a.col_idx, a.vals
            xr = np.random.default_rng(3).standard_normal(2 * n)
            t0 = time.perf_counter()
            for _ in range(3):
                O.matvec(rp, ci, va, xr)
            cpu_spmv = (time.perf_counter() - t0) / 3
            t0 = time.perf_counter()
            _, so = O.gmres(rp, ci, va, s.rhs, x0=x0, restart_m=30, tol=1e-10, max_total_iters=5,
                            precondition="jacobi")
            cpu_git = (time.perf_counter() - t0) / max(so.iterations, 1)
            cpu = {"kind": "port", "cores": 1, "spmv_ms": 1e3 * cpu_spmv, "gmres_ms_per_iteration": 1e3 * cpu_git,
                   "spmv_speedup": cpu_spmv / (ms.value / 1e3),
                   "sample": "3 oracle SpMVs and a 5-iteration GMRES(30)+Jacobi on the same matrix"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"error": str(exc)[:200]}
    return {"workload": "generate_box_mesh(80,80,79) cold system, 1,011,200 dofs", "cpu_baseline": cpu,
            "spmv": {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "frac_of_8TBs": ach / 8000.0, "us_per_launch": 1e3 * ms.value,
                     "bytes_per_launch": b_paired, "layout": "node-paired CSR (int32 col + double2 per slot)",
                     "kernel": "spmv_tma_pipe_kernel (TMA bulk-staged slot tiles, left-to-right rows)",
                     "thread_per_row_kernel_GBs": b_explicit / (ms_plain.value / 1e3) / 1e9,
                     "csr_equivalent_bytes": b_csr, "csr_equivalent_GBs": b_csr / (ms.value / 1e3) / 1e9,
                     "columns": (f"stencil classes ({ncls}; computed, values-only TMA stream)" if cls_on
                                 else "explicit int32 columns"),
                     "explicit_columns_equivalent_GBs": b_explicit / (ms.value / 1e3) / 1e9,
                     "l2": "flushed (256 MB write) before every timed launch", "peak_source": peak_src,
                     "back_to_back": {"launches": 1000, "us_per_launch": 1e3 * ms_b2b.value,
                                      "achieved": b_paired / (ms_b2b.value / 1e3) / 1e9,
                                      "frac": b_paired / (ms_b2b.value / 1e3) / 1e9 / hbm_peak,
                                      "us_per_launch_without_pdl": 1e3 * ms_b2b_plain.value,
                                      "dram_bytes_per_launch": b2b_dram,
                                      "dram_source": "committed ncu capture of launches inside such a chain "
                                                     "(profiles/r1k_spmv_c3_back_to_back_ncu.txt), not this run",
                                      "dram_GBs": (b2b_dram / (ms_b2b.value / 1e3) / 1e9) if b2b_dram else None,
                                      "dram_frac": (b2b_dram / (ms_b2b.value / 1e3) / 1e9 / hbm_peak)
                                      if b2b_dram else None,
                                      "protocol": "SURVEY 8(d) C3: 1,000 back-to-back SpMVs; the 137 MB matrix "
                                                  "stream exceeds the 126 MB L2, x (8 MB) stays L2-resident",
                                      "note": "no flush between launches; programmatic dependent launch streams "
                                              "a launch's first tiles while the previous one drains; DRAM bytes per "
                                              "launch from ncu inside such a chain "
                                              "(profiles/r1k_spmv_c3_back_to_back_ncu.txt)"}},
            "explicit_columns": expl,
            "pcg_cold_solve": {"l2": "flushed before the solve; iterations back to back",
                               "engine": {4: "kernel-per-phase (kp_spmv + kp_update)",
                                          3: "persistent TMA-streaming PCG"}.get(mode, str(mode)),
                               "bytes_per_iteration": it_bytes,
                               "iterations": st.iterations, "device_ms": st.device_ms,
                               "us_per_iteration": 1e3 * st.device_ms / max(st.iterations, 1),
                               "achieved_GBs": solve_ach, "frac": solve_ach / hbm_peak,
                               "final_relative_residual": st.final_relative_residual}}


def main():
    args = parse()
    if args.ref_worker:
        print(json.dumps(ref_worker(json.loads(args.ref_worker))), flush=True)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
