"""Full-size (2^30 packets over 2^32) checks without the CPU oracle, which cannot hold
these sizes (SURVEY.md 8(c) size-independent properties):

* the MSD + grouping path and the independent LSD onesweep path (NMX_PATH=lsd)
  give identical statistics -- at 2^30 the dense levels leave 2048 addresses per
  bucket, so the grouping kernels run their direct source / destination slots;
* relabeling invariance: complementing every address is a bijection of the
  address space, so all nine statistics are unchanged -- and with zeros injected
  first, the all-ones source and destination (the last slot of the last group)
  carry real traffic.
"""

import os

import pytest

pytestmark = pytest.mark.gpu

N = 1 << 30
SPACE = 1 << 32


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


def _both_paths(lib, s, d):
    msd = lib.stats9(s, d, None, SPACE)
    os.environ["NMX_PATH"] = "lsd"
    try:
        lsd = lib.stats9(s, d, None, SPACE)
    finally:
        del os.environ["NMX_PATH"]
    return msd, lsd


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_full_size_paths_and_relabeling(lib, kind):
    import torch

    from paper_2510_14050_b200.distributed import as_i32_tensor

    ds, dd = lib.DeviceArray(N), lib.DeviceArray(N)
    try:
        lib.generate(lib.GEN_UNIFORM if kind == "uniform" else lib.GEN_POWERLAW, 11, 0, N, SPACE, ds, dd)
        torch.cuda.synchronize()
        s, d = as_i32_tensor(ds, 0), as_i32_tensor(dd, 0)
        msd, lsd = _both_paths(lib, s, d)
        assert msd == lsd
        assert msd[0] == N

        # zeros injected (a hot source, a hot destination, one repeated link), then
        # every address complemented: 0 -> 0xFFFFFFFF
        s2, d2 = s.clone(), d.clone()
        s2[:5000] = 0
        d2[3000:9000] = 0
        s2 = torch.bitwise_not(s2)
        d2 = torch.bitwise_not(d2)
        torch.cuda.synchronize()
        inj_msd, inj_lsd = _both_paths(lib, s2, d2)
        assert inj_msd == inj_lsd
        # complementing back is the same relabeling: statistics unchanged
        s3, d3 = torch.bitwise_not(s2), torch.bitwise_not(d2)
        torch.cuda.synchronize()
        assert lib.stats9(s3, d3, None, SPACE) == inj_msd
        del s2, d2, s3, d3
    finally:
        ds.close()
        dd.close()
        torch.cuda.empty_cache()


def _full_golden(name):
    import json
    from pathlib import Path

    g = json.loads((Path(__file__).resolve().parent / "golden" / "full_size.json").read_text())
    return tuple(g["cases"][name]["stats9"])


@pytest.mark.parametrize("name", ["cfg3_seed7", "cfg3_seed11", "cfg4_seed7", "cfg4_seed11"])
def test_full_size_equals_chunked_oracle(lib, name):
    """N1: bit-exact nine statistics at 2^30 packets over 2^32 against the bounded-RAM
    chunked CPU oracle (oracle/nmx_oracle.c -> tests/golden/full_size.json), on the
    device path and the host (pinned, streamed) path."""
    import torch

    kind = lib.GEN_UNIFORM if name.startswith("cfg3") else lib.GEN_POWERLAW
    seed = int(name.split("seed")[1])
    want = _full_golden(name)
    ds, dd = lib.DeviceArray(N), lib.DeviceArray(N)
    try:
        lib.generate(kind, seed, 0, N, SPACE, ds, dd)
        assert lib.stats9(ds, dd, None, SPACE) == want
        if name == "cfg3_seed7":
            hs, hd = lib.PinnedArray(N), lib.PinnedArray(N)
            try:
                hs.array[:] = ds.download()
                hd.array[:] = dd.download()
                assert lib.stats9(hs.array, hd.array, None, SPACE) == want
            finally:
                hs.close()
                hd.close()
    finally:
        ds.close()
        dd.close()
        torch.cuda.empty_cache()
