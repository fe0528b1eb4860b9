"""libnmx.so loads without a GPU and exports every symbol include/nmx.h declares;
the product fails loudly (no CPU fallback) when no device is visible."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    text = (ROOT / "include" / "nmx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nmx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = _declared()
    for must in ("nmx_create", "nmx_stats9_device", "nmx_stats9_host", "nmx_window_stats9_host", "nmx_reduce_i64",
                 "nmx_coo_build", "nmx_flat_build", "nmx_partition_packets", "nmx_shard_rows", "nmx_shard_cols"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2510_14050_b200 import _lib

    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(_lib.SIGNATURES), "ctypes signatures out of sync with include/nmx.h"
    assert lib.nmx_version() >= 1


def _has_gpu():
    from paper_2510_14050_b200 import _lib

    return _lib.device_count() > 0


def test_fails_loudly_without_a_device():
    if _has_gpu():
        pytest.skip("a CUDA device is visible")
    from paper_2510_14050_b200 import NativeUnavailable, _lib

    with pytest.raises(NativeUnavailable):
        _lib.stats9(np.zeros(4, np.uint32), np.zeros(4, np.uint32), None, 16)


def test_sass_is_sm100a():
    import subprocess

    so = ROOT / "paper_2510_14050_b200" / "libnmx.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
