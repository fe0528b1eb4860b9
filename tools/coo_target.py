"""One device COO build (coo_from_packets) of 2^LOG2N uniform packets (target for ncu)."""
import sys
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib, coo

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(_lib.GEN_UNIFORM, 7, 0, n, 1 << 32, ds, dd)
for _ in range(reps):
    m = coo.coo_from_packets(ds, dd)
    print(m.nnz, _lib.context(0).last_timing())
    m.close()
