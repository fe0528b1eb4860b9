"""One cfg3-style stats9 call on device-resident packets (developer tool for ncu captures):
python tools/one_call.py [log2n] [kind]"""
import sys
sys.path.insert(0, ".")
from paper_2510_14050_b200 import _lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
kind = _lib.GEN_POWERLAW if len(sys.argv) > 2 and sys.argv[2] == "powerlaw" else _lib.GEN_UNIFORM
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
_lib.generate(kind, 7, 0, n, 1 << 32, ds, dd)
_lib.context(0)
print(_lib.stats9(ds, dd, None, 1 << 32))
