"""Seeded random configurations on the GPU against the packed-key oracle
(SURVEY.md 8(c)): sizes across the MSD path's range (2^16 up), address widths from 11 to
32 bits (direct and hashed grouping, light and heavy buckets), invalid packets,
device, host-chunked and streamed entry points."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1 << 16, (1 << 23) + 1))
    bits = int(rng.integers(11, 33))
    space = 1 << bits
    law = "powerlaw" if seed % 2 else "uniform"
    g = orc.gen_powerlaw if law == "powerlaw" else orc.gen_uniform
    s, d = g(seed, 0, n, space)
    s, d = s.copy(), d.copy()
    if seed % 3 == 0:  # a hot link and a hot destination on top
        k = n // 20
        s[:k] = s[0]
        d[:k] = d[1]
        d[k:2 * k] = d[2]
    v = rng.random(n) > 0.2 if seed % 4 == 1 else None
    return s, d, v, space


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("NMX_RANDOM_CASES", "16"))))
def test_random_configuration(lib, seed):
    s, d, v, space = _case(seed)
    want = orc.stats9_packed(s, d, v)
    if seed % 3 == 1:  # streamed windows of uneven length
        cut = [0, len(s) // 3, len(s) // 3 + 12345, len(s)]
        wins = [(s[a:b], d[a:b]) + ((v[a:b],) if v is not None else ()) for a, b in zip(cut, cut[1:])]
        assert lib.stream_stats9(wins, space) == want
    elif seed % 3 == 2 and v is None:  # device-resident columns
        ds, dd = lib.DeviceArray(len(s)), lib.DeviceArray(len(s))
        ds.upload(s)
        dd.upload(d)
        assert lib.stats9(ds, dd, None, space) == want
    else:
        assert lib.stats9(s, d, v, space) == want
