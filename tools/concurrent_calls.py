"""Do two independent stats9 calls overlap usefully on one B200? (developer tool: the
kernels are bound by different units -- scatters by the LSU data pipe, the grouping
kernels by issue -- so concurrent calls on two contexts / streams would show it)
python tools/concurrent_calls.py [log2n] [reps]"""
import sys, threading, time
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 29
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 1 << lg
ctxs = [_lib.Context(0), _lib.Context(0)]
arrs = []
for k in range(2):
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    _lib.generate(_lib.GEN_UNIFORM, 7 + k, 0, n, 1 << 32, ds, dd)
    arrs.append((ds, dd))

def call(k, out):
    with _lib.using(ctxs[k]):
        out[k] = _lib.stats9(arrs[k][0], arrs[k][1], None, 1 << 32)

res = [None, None]
for k in range(2):
    call(k, res)  # warm-up: workspaces grown
want = list(res)
for mode in ("sequential", "concurrent", "sequential", "concurrent"):
    best = 1e9
    for _ in range(reps):
        res = [None, None]
        t0 = time.perf_counter()
        if mode == "sequential":
            call(0, res); call(1, res)
        else:
            th = [threading.Thread(target=call, args=(k, res)) for k in range(2)]
            [t.start() for t in th]; [t.join() for t in th]
        dt = time.perf_counter() - t0
        assert res == want, (res, want)
        best = min(best, dt)
    print(f"{mode:10s} 2 x 2^{lg}: {best * 1e3:8.2f} ms ({2 * n / best / 1e9:.2f} Gpkt/s)", flush=True)
