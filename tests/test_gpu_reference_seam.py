"""The drop-in, proven with the REAL reference on the B200.

The unmodified reference package (rafem 0.1.0) is staged into
baseline/_ref by scripts/stage_reference.sh (build() runs it when
/root/reference is present; baseline/_ref travels to the GPU box).  Here:

* the reference's own ``rafem.fem.run_simulation`` runs with
  ``plugin.install()`` routing its corrector's ``assemble_global`` /
  ``solve`` (fem.py:47-48, 492, 501) to the device path — A40 (configs[0])
  and B900 (configs[1]) — and must reproduce the reference's golden runs:
  identical trajectory, final-step fields within 1e-6 (every step at
  1e-12 against the 1e-12 golden), PSNR above the 1e-5 noise control;
* the reference's own test suite (test_fem, test_acceptance, test_solver,
  ...) runs with the seam installed through tests/seam_plugin.py.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden
from test_gpu_assembly_sim import _compare_run

pytestmark = pytest.mark.gpu

REF = os.path.join(ROOT, "baseline", "_ref")
needs_ref = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rafem")),
                               reason="reference not staged (scripts/stage_reference.sh)")


class _Rec:
    def __init__(self, d, i):
        self.time, self.dt, self.corrector_iters = float(d["time"][i]), float(d["dt"][i]), int(d["corrector_iters"][i])
        self.T, self.V = d["T"][i], d["V"][i]


def _seam_run(tmp_path, dims, total, solver="gmres", tol=1e-10):
    out = str(tmp_path / f"seam_{solver}_{tol:g}.npz")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "seam_runs.py"), out, *map(str, dims), str(total),
                        solver, str(tol)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = np.load(out)
    return [_Rec(d, i) for i in range(len(d["time"]))], d


@needs_ref
@pytest.mark.parametrize("solver", ["gmres", "pcg"])
def test_reference_run_simulation_A40_through_seam(tmp_path, solver):
    recs, d = _seam_run(tmp_path, (15, 15, 16), 40.0, solver)
    assert d["seam"][0] == d["summary"][1] and d["seam"][1] == d["summary"][1]  # every pass on the device
    assert d["seam"][2] == 0
    _compare_run(recs, golden("run_A40_1e-10"), 1e-6, every_step=False)


@needs_ref
@pytest.mark.parametrize("solver", ["gmres", "pcg"])
def test_reference_run_simulation_B900_through_seam(tmp_path, solver):
    g = golden("run_B900_1e-10")
    recs, d = _seam_run(tmp_path, (20, 20, 21), 900.0, solver)
    assert int(d["summary"][0]) == 96 and int(d["summary"][1]) == int(g["summary"][1])
    assert d["seam"][1] == d["summary"][1] and d["seam"][2] == 0
    _compare_run(recs, g, 1e-6, every_step=False)
    recs12, _ = _seam_run(tmp_path, (20, 20, 21), 900.0, solver, 1e-12)
    _compare_run(recs12, golden("run_B900_1e-12"), 1e-6, every_step=True)


@needs_ref
def test_reference_test_suite_with_seam_installed():
    """The reference's own tests, with its fem seam on the device path.
    Deselected: the --plot CLI tests (matplotlib is not in the image; they
    fail without the seam too)."""
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests")]))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "seam_plugin",
                        "-k", "not plot", os.path.join(REF, "rafem_tests")],
                       capture_output=True, text=True, env=env, cwd=os.path.join(REF, "rafem_tests"), timeout=1800)
    tail = r.stdout[-6000:]
    print(tail)
    assert r.returncode == 0, tail + r.stderr[-2000:]
    seam = [ln for ln in r.stdout.splitlines() if ln.startswith("SEAM ")]
    assert seam, tail
    fields = dict(kv.split("=", 1) for kv in seam[-1].split()[1:] if "=" in kv and not kv.startswith("backends"))
    assert os.path.realpath(fields["rafem"]).startswith(os.path.realpath(REF))
    assert int(fields["assemble"]) > 100 and int(fields["solve_device"]) > 100
