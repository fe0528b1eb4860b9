"""One stats9 call on device-resident synthetic packets (target for ncu).

    python tools/profile_target.py LOG2N [powerlaw] [reps=R]
"""
import sys
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib

kind = _lib.GEN_POWERLAW if "powerlaw" in sys.argv else _lib.GEN_UNIFORM
lg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 28
reps = next((int(a[5:]) for a in sys.argv if a.startswith("reps=")), 2)
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(kind, 7, 0, n, 1 << 32, ds, dd)
for _ in range(reps):
    print(_lib.stats9(ds, dd, None, 1 << 32), _lib.context(0).last_timing())
