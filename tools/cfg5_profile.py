"""Break down the streamed cfg5 path (developer tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_14050_b200 import _lib, coo as nc

w = 1 << 28
nwin = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = _lib.context(0)
ds, dd = _lib.DeviceArray(w), _lib.DeviceArray(w)
pins = []
for k in range(2):
    _lib.generate(_lib.GEN_UNIFORM, 7, k * w, w, 1 << 32, ds, dd)
    ps, pd = _lib.PinnedArray(w), _lib.PinnedArray(w)
    ps.array[:] = ds.download(); pd.array[:] = dd.download()
    pins.append((ps, pd))
nc.reserve(64 << 30)
def T(f, *a):
    t0 = time.perf_counter(); r = f(*a); return r, (time.perf_counter() - t0) * 1e3
_, t = T(lambda: ds.upload(pins[0][0].array)); print(f"H2D one column 1 GiB: {t:.1f} ms", flush=True)
for rep in range(2):
    c1, t = T(nc.coo_from_packets, ds, dd); print(f"build window: {t:.1f} ms nnz={c1.nnz} {ctx.last_timing()['stages_ms']}", flush=True)
c2, _ = T(nc.coo_from_packets, ds, dd)
m, t = T(nc.merge_add, c1, c2); print(f"merge 2x2^28: {t:.1f} ms", flush=True)
m2, t = T(nc.merge_add, m, m); print(f"merge 2x{m.nnz}: {t:.1f} ms", flush=True)
s, t = T(m2.stats9); print(f"stats9 of {m2.nnz}: {t:.1f} ms {ctx.last_timing()['stages_ms']}", flush=True)
views = [(pins[k % 2][0].array, pins[k % 2][1].array) for k in range(nwin)]
r, t = T(nc.stream_stats9_pinned, views); print(f"stream {nwin} windows: {t:.1f} ms", flush=True)
