"""Merge-add of two 2^27-link device COOs with a given libnmx build (A/B target for ncu):
python tools/merge_ab.py [path/to/libnmx.so]"""
import sys
sys.path.insert(0, ".")
from pathlib import Path
from paper_2510_14050_b200 import _lib, coo

if len(sys.argv) > 1:
    _lib.LIB_PATH = Path(sys.argv[1])
lg = 27
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
parts = []
for k in range(2):
    _lib.generate(_lib.GEN_UNIFORM, 7, k * n, n, 1 << 32, ds, dd)
    parts.append(coo.coo_from_packets(ds, dd))
for _ in range(3):
    m = coo.merge_add(parts[0], parts[1])
    print(m.nnz, m.stats9())
    m.close()
