"""Cold single-launch SpMV with and without the per-tile L2 prefetch of x
(RAFEM_XPF=1), a few tile configurations, at C3 (and C4 when asked).

    python scripts/spmv_xpf_probe.py [nx ny nz]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    dims = tuple(map(int, sys.argv[1:4])) if len(sys.argv) >= 4 else (80, 80, 79)
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200.assembly import DeviceMesh, SystemHandle
    dm = DeviceMesh.from_box(*dims)
    h = SystemHandle(dm)
    n = dm.node_count
    p = nat.AssembleParams()
    p.dt, p.applied_voltage, p.boundary_temp, p.apply_constraints, p.equilibrate = 0.5, 25.0, 37.0, 1, 1
    t = np.full(n, 37.0)
    v = np.zeros(n)
    sc, bad = C.c_double(), C.c_int64()
    nat.check(nat.lib().rafem_assemble(h.handle, nat.ptr(t), nat.ptr(v), nat.ptr(t), C.byref(p), C.byref(sc),
                                       C.byref(bad)), "asm")
    S = dm.slots
    B = 16 * S + n + 4 * (n + 1) + 32 * n
    x = np.random.default_rng(1).standard_normal(2 * n)
    ys = {}
    for cfg in ["", "128,3,1,2", "256,2,1,1", "192,3,1,1", "128,4,1,2"]:
        for xpf in ("0", "1"):
            os.environ["RAFEM_XPF"] = xpf
            if cfg:
                os.environ["RAFEM_SPMV_CFG"] = cfg
            else:
                os.environ.pop("RAFEM_SPMV_CFG", None)
            ms = C.c_double()
            rc = nat.lib().rafem_system_spmv_bench(h.handle, 30, 1, C.byref(ms))
            if rc:
                print(cfg or "default", "xpf", xpf, "rc", rc)
                continue
            y = np.empty(2 * n)
            nat.check(nat.lib().rafem_system_spmv(h.handle, nat.ptr(x), nat.ptr(y)), "spmv")
            ys[(cfg, xpf)] = y
            print(f"{cfg or 'default':12s} xpf={xpf}: {1e3 * ms.value:7.2f} us  {B / ms.value / 1e6:7.0f} GB/s "
                  f"({B / ms.value / 1e6 / 6538.3:.3f} of measured)", flush=True)
    ref = next(iter(ys.values()))
    print("all bitwise equal:", all(np.array_equal(ref, y) for y in ys.values()))


if __name__ == "__main__":
    main()
