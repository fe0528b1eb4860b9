"""Repeated small stats9 calls on device-resident packets (ncu target for the small-call path)."""
import sys
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 17
space = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(_lib.GEN_UNIFORM, 7, 0, n, space, ds, dd)
for _ in range(3):
    print(_lib.stats9(ds, dd, None, space), _lib.context(0).last_timing())
