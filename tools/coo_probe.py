"""Developer probe: COO build / merge / stats9 pieces at 2^lg (kernel launch list target)."""
import sys, time
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib, coo as nc

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << lg
ctx = _lib.context(0)
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(_lib.GEN_UNIFORM, 7, 0, n, 1 << 32, ds, dd)
c1 = nc.coo_from_packets(ds, dd)
_lib.generate(_lib.GEN_UNIFORM, 7, n, n, 1 << 32, ds, dd)
c2 = nc.coo_from_packets(ds, dd)
for rep in range(2):
    t0 = time.perf_counter(); m = nc.merge_add(c1, c2); t1 = time.perf_counter()
    s = m.stats9(); t2 = time.perf_counter()
    print(f"merge {(t1-t0)*1e3:.1f} ms nnz={m.nnz}; stats9 {(t2-t1)*1e3:.1f} ms {ctx.last_timing()['stages_ms']}", flush=True)
    m.close()
