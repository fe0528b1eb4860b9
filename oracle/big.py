"""ctypes binding of oracle/nmx_oracle.c -- TEST INFRASTRUCTURE ONLY.

The bounded-RAM chunked packed-key oracle (restating traffic.py:197-292 +
analytics.py:89-106 of /root/reference/pkg/src/netmeter, see the C header) for
sizes the dense reference and the in-memory numpy restatement cannot hold
(SURVEY.md 8(c) "Large sizes"). Only tests/, tools/ and oracle/make_full_size.py
load it; the product package never does.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "nmx_oracle.c"
LIB = HERE / "_build" / "libnmx_oracle.so"
UNIFORM, POWERLAW = 0, 1
_lib = None


def build() -> Path:
    LIB.parent.mkdir(exist_ok=True)
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-o", str(LIB), str(SRC)],
                       check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        u64, i64p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_int64)
        lib.nmx_oracle_stats9_gen.argtypes = [ctypes.c_int, u64, u64, u64, u64, ctypes.c_int, i64p]
        lib.nmx_oracle_stats9_pairs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, u64,
                                                ctypes.c_int, i64p]
        lib.nmx_oracle_generate.argtypes = [ctypes.c_int, u64, u64, u64, u64, ctypes.c_void_p, ctypes.c_void_p]
        _lib = lib
    return _lib


def _bucket_bits(n: int) -> int:
    # about 2^26 keys (512 MiB) per bucket
    return max(0, min(12, (max(n, 1) - 1).bit_length() - 26))


def stats9_gen(kind: int, seed: int, offset: int, n: int, space: int = 1 << 32, bucket_bits: int | None = None):
    out = (ctypes.c_int64 * 9)()
    bb = _bucket_bits(n) if bucket_bits is None else bucket_bits
    rc = load().nmx_oracle_stats9_gen(kind, seed, offset, n, space, bb, out)
    if rc:
        raise RuntimeError(f"nmx_oracle_stats9_gen failed: {rc}")
    return tuple(int(v) for v in out)


def stats9_pairs(src, dst, valid=None, bucket_bits: int | None = None):
    s = np.ascontiguousarray(src, dtype=np.uint32)
    d = np.ascontiguousarray(dst, dtype=np.uint32)
    v = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
    out = (ctypes.c_int64 * 9)()
    bb = _bucket_bits(len(s)) if bucket_bits is None else bucket_bits
    rc = load().nmx_oracle_stats9_pairs(s.ctypes.data, d.ctypes.data, None if v is None else v.ctypes.data,
                                        len(s), bb, out)
    if rc:
        raise RuntimeError(f"nmx_oracle_stats9_pairs failed: {rc}")
    return tuple(int(x) for x in out)


def generate(kind: int, seed: int, offset: int, n: int, space: int = 1 << 32):
    s = np.empty(n, np.uint32)
    d = np.empty(n, np.uint32)
    rc = load().nmx_oracle_generate(kind, seed, offset, n, space, s.ctypes.data, d.ctypes.data)
    if rc:
        raise RuntimeError(f"nmx_oracle_generate failed: {rc}")
    return s, d
