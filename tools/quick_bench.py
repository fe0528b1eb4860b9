"""Quick device timing sweep of the stats9 hot path (developer tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_14050_b200 import _lib

def run(kind, lg, space, reps=5):
    n = 1 << lg
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    _lib.generate(kind, 7, 0, n, space, ds, dd)
    ctx = _lib.context(0)
    best = None
    for r in range(reps):
        t0 = time.perf_counter()
        st = _lib.stats9(ds, dd, None, space)
        wall = time.perf_counter() - t0
        t = ctx.last_timing()
        if best is None or t["total_ms"] < best[0]["total_ms"]:
            best = (t, wall)
    t, wall = best
    print(f"kind={kind} n=2^{lg} space={space}: dev {t['total_ms']:.3f} ms  sort {t['sort_ms']:.3f} ms "
          f"({t['sort_launches']} passes) wall {wall*1e3:.2f} ms  -> {n/t['total_ms']/1e6:.2f} Gpkt/s  "
          f"launches={t['kernel_launches']} stats={st}", flush=True)
    ds.close(); dd.close()

for lg in (17, 20, 23, 26, 28, 30):
    run(_lib.GEN_UNIFORM, lg, 1 << 32)
for lg in (23, 26, 30):
    run(_lib.GEN_POWERLAW, lg, 1 << 32)
run(_lib.GEN_UNIFORM, 23, 1 << 24)
