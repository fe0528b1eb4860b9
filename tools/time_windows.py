"""Live timing of per-window statistics (nmx_window_stats9_device) and of a device COO
build (developer tool): python tools/time_windows.py"""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2510_14050_b200 import _lib, coo

ctx = _lib.context(0)
for lg, wlg, space in ((23, 17, 1 << 24), (26, 20, 1 << 28), (28, 22, 1 << 32)):
    n = 1 << lg
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    _lib.generate(_lib.GEN_UNIFORM, 7, 0, n, space, ds, dd)
    best, bt = None, None
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w = _lib.window_stats9(ds, dd, None, space, 1 << wlg)
        t = time.perf_counter() - t0
        if best is None or t < best:
            best, bt = t, ctx.last_timing()
    print(f"windows 2^{lg} / 2^{wlg} over {space}: {best * 1e3:.3f} ms wall, device {bt['total_ms']:.3f} ms "
          f"({n / best / 1e9:.2f} Gpkt/s), dom {bt['dom_name']} {bt['dom_ms'] / max(bt['dom_launches'], 1):.3f} ms x{bt['dom_launches']}, "
          f"launches {bt['kernel_launches']}, rows {len(w)}", flush=True)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = coo.coo_from_packets(ds, dd)
        nnz = m.nnz
        ts.append(time.perf_counter() - t0)
        m.close()
    print(f"coo build 2^{lg}: {min(ts) * 1e3:.3f} ms wall (nnz {nnz})", flush=True)
    ds.close(); dd.close()
