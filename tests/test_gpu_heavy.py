"""GPU parity for heavy hitters on the MSD path (n >= 2^20): buckets larger than a
shared-memory group go through the segmented MSD levels (csrc/nmx_seg.cuh) --
whole-source levels, single-source levels with partial fan-out accumulated in the
global source table, and the count-only final level (one link / one destination
per child). Bit-exact against the packed-key oracle."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu

N = 1 << 20


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


def _check(lib, s, d, space, v=None):
    s = np.asarray(s, np.uint32)
    d = np.asarray(d, np.uint32)
    assert lib.stats9(s, d, v, space) == orc.stats9_packed(s, d, v)


def test_one_source_random_destinations(lib):
    rng = np.random.default_rng(1)
    s = np.full(N, 123456789, np.uint32)
    d = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
    _check(lib, s, d, 1 << 32)


def test_one_source_few_destinations(lib):
    rng = np.random.default_rng(2)
    s = np.full(N, 7, np.uint32)
    d = rng.integers(0, 3000, N).astype(np.uint32)  # long duplicate runs per link
    _check(lib, s, d, 1 << 32)


def test_single_link(lib):
    s = np.full(N, 0xFFFFFFFF, np.uint32)
    d = np.full(N, 0xFFFFFFFF, np.uint32)
    _check(lib, s, d, 1 << 32)
    _check(lib, np.zeros(N, np.uint32), np.zeros(N, np.uint32), 1 << 32)


def test_one_destination_many_sources(lib):
    rng = np.random.default_rng(3)
    s = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
    d = np.full(N, 99, np.uint32)
    _check(lib, s, d, 1 << 32)


def test_all_ones_source_and_destination_heavy(lib):
    # the all-ones source / destination use reserved slots (src + 1 overflows)
    rng = np.random.default_rng(4)
    s = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(0, 1 << 32, N, dtype=np.uint64).astype(np.uint32)
    s[: N // 3] = 0xFFFFFFFF
    d[N // 3 : 2 * N // 3] = 0xFFFFFFFF
    d[: N // 10] = rng.integers(0, 50, N // 10).astype(np.uint32)
    _check(lib, s, d, 1 << 32)


def test_heavy_mixture_with_invalid(lib):
    rng = np.random.default_rng(5)
    n = 3 * N // 2 + 777
    s, d = orc.gen_powerlaw(77, 0, n, 1 << 32)
    s = s.copy()
    d = d.copy()
    hot = rng.integers(0, 1 << 32, 6, dtype=np.uint64).astype(np.uint32)
    pick = rng.integers(0, 6, n // 4)
    s[: n // 4] = hot[pick]
    d[n // 8 : n // 4] = hot[(pick[n // 8 :] + 1) % 6]
    v = rng.random(n) > 0.1
    _check(lib, s, d, 1 << 32, v)


@pytest.mark.parametrize("bits", [11, 12, 16, 21, 26])
def test_powerlaw_small_spaces(lib, bits):
    # bits == 11 at n = 2^20: the dense levels already isolate single sources
    space = 1 << bits
    s, d = orc.gen_powerlaw(9, 0, N, space)
    _check(lib, s, d, space)


@pytest.mark.parametrize("seed", [1, 2])
def test_powerlaw_2_24(lib, seed):
    s, d = orc.gen_powerlaw(seed, 0, 1 << 24, 1 << 32)
    _check(lib, s, d, 1 << 32)


def test_skewed_uniform_blend(lib):
    # many medium sources (a few thousand packets each) spread over all buckets
    rng = np.random.default_rng(6)
    n = 1 << 22
    srcs = rng.integers(0, 1 << 32, 900, dtype=np.uint64).astype(np.uint32)
    s = srcs[rng.integers(0, 900, n)]
    d = rng.integers(0, 1 << 20, n).astype(np.uint32)
    _check(lib, s, d, 1 << 32)


def test_u8_count_escapes_on_the_column_path(lib):
    # links with 255 / 256 / 257 / 1000 / 65536 packets: counts >= 256 leave the
    # column path's u8 counts through the destination table (incl. dst 0xFFFFFFFF
    # and a destination that only receives escaped links)
    rng = np.random.default_rng(8)
    parts_s, parts_d = [], []
    for i, c in enumerate([255, 256, 257, 1000, 65536, 300, 299]):
        parts_s.append(np.full(c, 1000 + i, np.uint32))
        parts_d.append(np.full(c, 77 if i < 5 else 0xFFFFFFFF, np.uint32))
    parts_s.append(np.full(400, 5, np.uint32))
    parts_d.append(np.full(400, 123456, np.uint32))  # only escaped links
    parts_s.append(np.full(600, 6, np.uint32))
    parts_d.append(np.full(600, 123456, np.uint32))
    n_bg = (1 << 21) - sum(len(x) for x in parts_s)
    parts_s.append(rng.integers(0, 1 << 32, n_bg, dtype=np.uint64).astype(np.uint32))
    parts_d.append(rng.integers(0, 1 << 32, n_bg, dtype=np.uint64).astype(np.uint32))
    s, d = np.concatenate(parts_s), np.concatenate(parts_d)
    perm = rng.permutation(len(s))
    _check(lib, s[perm], d[perm], 1 << 32)


@pytest.mark.parametrize("logn,bits,law", [(25, 27, "uniform"), (26, 28, "powerlaw"), (22, 12, "powerlaw"),
                                           (23, 20, "uniform")])
def test_direct_source_and_destination_slots(lib, logn, bits, law):
    # groups whose buckets span few addresses index sources (and destinations)
    # directly: 2^(bits - D) addresses per bucket (D = logn - 9; D > bits at 2^22 / 2^12)
    n = 1 << logn
    space = 1 << bits
    if law == "uniform":
        rng = np.random.default_rng(logn + bits)
        s = rng.integers(0, space, n, dtype=np.uint64).astype(np.uint32)
        d = rng.integers(0, space, n, dtype=np.uint64).astype(np.uint32)
        s[:1000] = space - 1  # the last source / destination of the space
        d[500:1500] = space - 1
    else:
        s, d = orc.gen_powerlaw(logn, 0, n, space)
    _check(lib, s, d, space)


def test_direct_destination_slots_with_large_counts(lib):
    # direct destination slots (2^25 packets over 2^27: 2048 destinations per bucket)
    # pack fan-in with counts < 512 in one word; counts >= 512 take the second
    # word: a destination with 400 links of 511 packets (its bucket stays light,
    # ~900 entries), one with counts around and far above 512
    rng = np.random.default_rng(12)
    space = 1 << 27
    n_bg = 1 << 25
    s = [rng.integers(0, space, n_bg, dtype=np.uint64).astype(np.uint32)]
    d = [rng.integers(0, space, n_bg, dtype=np.uint64).astype(np.uint32)]
    x, y = 123_456_789 % space, 98_765_432 % space
    srcs = rng.choice(space, 400, replace=False).astype(np.uint32)
    s.append(np.repeat(srcs, 511))
    d.append(np.full(400 * 511, x, np.uint32))
    for i, c in enumerate([512, 513, 1000, 5000, 100_000, 511, 1]):
        s.append(np.full(c, 7 + i, np.uint32))
        d.append(np.full(c, y, np.uint32))
    s, d = np.concatenate(s), np.concatenate(d)
    perm = rng.permutation(len(s))
    _check(lib, s[perm], d[perm], space)
