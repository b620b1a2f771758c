"""Assembly A/B at benchmark sizes: fused element+fill with the pipelined
half-warp fill (default) vs the same fill without the row pipeline
(RAFEM_FILL_PIPE=0), the warp fill (RAFEM_HALF_FILL=0) and the element
kernel + contributor-list fill (RAFEM_FUSED_FILL=0).  Times one
device-field assembly (rafem_sl_assemble_partial + rafem_assemble_finish,
incl. the diagonal-sum read-back) and checks the two paths bitwise.

    python scripts/asm_probe.py [NX NY NZ] [reps]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    dims = tuple(map(int, sys.argv[1:4])) if len(sys.argv) >= 4 else (200, 200, 200)
    reps = int(sys.argv[4]) if len(sys.argv) >= 5 else 5
    import torch
    from paper_2409_13036_b200 import SimConfig
    from paper_2409_13036_b200 import _native as nat
    from paper_2409_13036_b200.assembly import DeviceMesh
    from paper_2409_13036_b200.shard import DeviceShardedSimulation, ShardedSystem
    L = nat.lib()
    dm = DeviceMesh.from_box(*dims)
    sh = ShardedSystem.from_device_mesh(dm)
    loop = DeviceShardedSimulation(sh)
    nat.check(L.rafem_sl_init(loop.h, 37.0), "init")
    nat.check(L.rafem_sl_predict(loop.h, 0, 1.0, 0), "predict")
    p = sh.assemble_params(4.0, SimConfig())
    sums = np.zeros(2)
    bad = C.c_int64()
    out = {}
    for mode, half, pipe in (("1", "1", "1"), ("1", "1", "0"), ("1", "0", "1"), ("0", "1", "1"), ("1", "1", "1")):
        os.environ["RAFEM_FUSED_FILL"] = mode
        os.environ["RAFEM_HALF_FILL"] = half
        os.environ["RAFEM_FILL_PIPE"] = pipe
        mode = mode + half + pipe
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nat.check(L.rafem_sl_assemble_partial(loop.h, 4.0, nat.ptr(sums), C.byref(bad)), "asm")
            nat.check(L.rafem_assemble_finish(sh.h.handle, C.byref(p), 1.0), "finish")
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        vals = sh.h.download_vals()
        rhs = sh.h.rhs()
        out.setdefault(mode, (vals, rhs))
        print(f"fused,half,pipe={mode}: {dims} N={dm.node_count} M={dm.tet_count}: assembly {1e3 * min(ts):.2f} ms "
              f"(median {1e3 * sorted(ts)[len(ts) // 2]:.2f})", flush=True)
    for k in ("110", "101", "011"):
        same = np.array_equal(out["111"][0], out[k][0]) and np.array_equal(out["111"][1], out[k][1])
        print(f"pipelined half-warp fill == {k} (fused, half, pipe) bitwise:", same)


if __name__ == "__main__":
    main()
