"""Developer probe: stats9 on device-generated packets at several sizes (crash bisection)."""
import sys
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib

kind = _lib.GEN_POWERLAW if "powerlaw" in sys.argv else _lib.GEN_UNIFORM
for lg in [int(a) for a in sys.argv[1:] if a.isdigit()]:
    n = 1 << lg
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    _lib.generate(kind, 7, 0, n, 1 << 32, ds, dd)
    print(lg, _lib.stats9(ds, dd, None, 1 << 32), _lib.context(0).last_timing()["stages_ms"], flush=True)
    ds.close(); dd.close()
