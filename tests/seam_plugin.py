"""pytest plugin (test infrastructure): run the REFERENCE's own test modules
— staged unmodified under baseline/_ref/rafem_tests by
scripts/stage_reference.sh — with rafem.fem's plug-in seam (fem.py:47-48,
492, 501) pointed at the B200 path before any test module imports it.

    PYTHONPATH=baseline/_ref:.:tests python -m pytest -p seam_plugin baseline/_ref/rafem_tests

RAFEM_SEAM_SOLVER=pcg serves "gmres" configurations with the device PCG
(plugin.install(solver="pcg")).  The terminal summary prints how many
assemblies and solves went through the device path.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    if ROOT not in sys.path:
        sys.path.insert(1, ROOT)
    import rafem.fem  # noqa: F401  (the staged reference)
    from paper_2409_13036_b200 import _native, plugin
    _native.context()  # fail loudly without the library or a device
    plugin.install("rafem.fem", solver=os.environ.get("RAFEM_SEAM_SOLVER") or None)


def pytest_terminal_summary(terminalreporter):
    import rafem
    from paper_2409_13036_b200 import _native, plugin
    c = plugin.counters
    terminalreporter.write_line(
        f"SEAM rafem={os.path.dirname(rafem.__file__)} assemble={c.assemble} solve_device={c.solve_device} "
        f"solve_passthrough={c.solve_passthrough} backends={c.backends} launches={_native.kernel_launches()}")
