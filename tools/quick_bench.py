"""Quick device timing sweep of the stats9 hot path (developer tool)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2510_14050_b200 import _lib

def run(kind, lg, space, reps=4):
    n = 1 << lg
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    _lib.generate(kind, 7, 0, n, space, ds, dd)
    ctx = _lib.context(0)
    best = None
    for r in range(reps):
        st = _lib.stats9(ds, dd, None, space)
        t = ctx.last_timing()
        if best is None or t["total_ms"] < best["total_ms"]:
            best = t
    t = best
    print(f"kind={kind} n=2^{lg} space={space}: dev {t['total_ms']:.3f} ms -> {n/t['total_ms']/1e6:.2f} Gpkt/s "
          f"stages={t['stages_ms']} launches={t['kernel_launches']} stats={st}", flush=True)
    ds.close(); dd.close()
    return st

lgs = [int(x) for x in sys.argv[1:]] or [20, 23, 26, 28, 30]
for lg in lgs:
    run(_lib.GEN_UNIFORM, lg, 1 << 32)
for lg in lgs:
    run(_lib.GEN_POWERLAW, lg, 1 << 32)
