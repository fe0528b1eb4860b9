"""Merge-add of two device COOs of 2^LOG2N links each (target for ncu)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2510_14050_b200 import _lib, coo

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << lg
ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
parts = []
for k in range(2):
    _lib.generate(_lib.GEN_UNIFORM, 7, k * n, n, 1 << 32, ds, dd)
    parts.append(coo.coo_from_packets(ds, dd))
for _ in range(2):
    m = coo.merge_add(parts[0], parts[1])
    print(m.nnz)
    m.close()
