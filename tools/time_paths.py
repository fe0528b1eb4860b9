"""Live timings of the LSD path (NMX_PATH=lsd, one onesweep pass class) and merge-add
(developer tool): python tools/time_paths.py [lsd_log2n] [merge_log2n]"""
import os, sys, time
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib, coo

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
mg = int(sys.argv[2]) if len(sys.argv) > 2 else 27
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(_lib.GEN_UNIFORM, 7, 0, n, 1 << 32, ds, dd)
ctx = _lib.context(0)
os.environ["NMX_PATH"] = "lsd"
best = None
for _ in range(4):
    st = _lib.stats9(ds, dd, None, 1 << 32)
    t = ctx.last_timing()
    if best is None or t["total_ms"] < best["total_ms"]:
        best = t
print(f"lsd 2^{lg}: total {best['total_ms']:.3f} ms, {best['dom_name']} {best['dom_ms'] / best['dom_launches']:.3f} ms/launch "
      f"x{best['dom_launches']} ({best['dom_bytes'] / best['dom_launches'] / (best['dom_ms'] / best['dom_launches']) / 1e6:.0f} GB/s) {st}", flush=True)
del os.environ["NMX_PATH"]
ds.close(); dd.close()
if not mg:
    sys.exit(0)
m = 1 << mg
ds, dd = _lib.DeviceArray(m), _lib.DeviceArray(m)
parts = []
for k in range(2):
    _lib.generate(_lib.GEN_UNIFORM, 7, k * m, m, 1 << 32, ds, dd)
    parts.append(coo.coo_from_packets(ds, dd))
ts = []
for _ in range(4):
    ctx.synchronize() if hasattr(ctx, "synchronize") else None
    t0 = time.perf_counter()
    r = coo.merge_add(parts[0], parts[1])
    nnz = r.nnz
    ts.append(time.perf_counter() - t0)
    r.close()
print(f"merge 2^{mg}+2^{mg}: best {min(ts) * 1e3:.3f} ms wall (nnz {nnz})", flush=True)
