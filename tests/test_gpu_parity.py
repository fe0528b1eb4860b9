"""GPU parity: libnmx.so (through its C ABI) vs the CPU oracle / golden vectors.

Bit-exact equality for every statistic (integer work)."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


def _pairs(case):
    p = np.array(case["pairs"], dtype=np.int64).reshape(-1, 2)
    valid = np.array(case.get("valid", [1] * len(p)), dtype=bool)
    return p[:, 0], p[:, 1], valid


@pytest.mark.parametrize("name", ["hand", "hand_other", "oracle_hand", "self_loops", "invalid_hand"])
def test_hand_vectors(lib, golden, name):
    case = golden["cases"][name]
    s, d, v = _pairs(case)
    space = int(max(s.max(), d.max())) + 1
    assert lib.stats9(s, d, v, space) == tuple(case["stats9"])


def test_empty_and_all_invalid(lib):
    e = np.zeros(0, np.uint32)
    assert lib.stats9(e, e, None, 16) == (0,) * 9
    s = np.arange(100, dtype=np.uint32) % 7
    assert lib.stats9(s, s, np.zeros(100, bool), 16) == (0,) * 9
    one = np.array([3], np.uint32)
    assert lib.stats9(one, one, None, 4) == (1, 1, 1, 1, 1, 1, 1, 1, 1)


def test_corpus(lib, golden):
    for c in golden["cases"]["corpus"]:
        s, d, v = orc.generate_packets(c["n"], c["space"], c["seed"], c["invalid_fraction"])
        assert lib.stats9(s, d, v, c["space"]) == tuple(c["stats9"]), c


@pytest.mark.parametrize("name", ["cfg1", "windows_small", "windows_invalid", "invariance"])
def test_generate_anonymize_cases(lib, golden, name):
    c = golden["cases"][name]
    s, d, v = orc.generate_packets(c["n"], c["space"], c["seed"], c["invalid_fraction"])
    space = c["space"]
    if c["anon_key"] is not None:
        s, d, space = orc.anonymize(s, d, c["anon_key"])
    assert lib.stats9(s, d, v, space) == tuple(c["stats9"])
    if "window" in c:
        got = lib.window_stats9(s, d, v, space, c["window"])
        assert got.tolist() == c["windows9"]


def test_cfg2_summed_and_windows(lib, golden):
    c = golden["cases"]["cfg2"]
    s, d, v = orc.generate_packets(c["n"], c["space"], c["seed"], c["invalid_fraction"])
    s, d, space = orc.anonymize(s, d, c["anon_key"])
    assert orc.checksum_u32(s) == c["src_sha"]
    assert lib.stats9(s, d, v, space) == tuple(c["stats9"])
    got = lib.window_stats9(s, d, v, space, c["window"])
    assert got.tolist() == c["windows9"]
    assert orc.to6(orc.totals9([tuple(r) for r in got.tolist()])) == tuple(c["totals6"])


def test_splitmix_cases(lib, golden):
    for name, c in golden["cases"]["splitmix"].items():
        gen = orc.gen_uniform if c["kind"] == "uniform" else orc.gen_powerlaw
        s, d = gen(c["seed"], 0, c["n"], c["space"])
        assert lib.stats9(s, d, None, c["space"]) == tuple(c["stats9"]), name


def test_device_generator_matches_oracle(lib):
    n = 1 << 20
    for kind, gen in ((lib.GEN_UNIFORM, orc.gen_uniform), (lib.GEN_POWERLAW, orc.gen_powerlaw)):
        for space in (1 << 32, 1000, 1 << 24):
            ds, dd = lib.DeviceArray(n), lib.DeviceArray(n)
            lib.generate(kind, 9, 12345, n, space, ds, dd)
            s, d = gen(9, 12345, n, space)
            assert np.array_equal(ds.download(), s) and np.array_equal(dd.download(), d)
            assert lib.stats9(ds, dd, None, space) == orc.stats9_packed(s, d)


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("lg,space", [(23, 1 << 32), (24, 1 << 20), (25, 1 << 32), (27, 1 << 20), (27, (1 << 30) + 7)])
def test_large_vs_packed_oracle(lib, kind, lg, space):
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = gen(5, 0, 1 << lg, space)
    assert lib.stats9(s, d, None, space) == orc.stats9_packed(s, d)


@pytest.mark.parametrize("case", ["hot_dst", "tiny_level1", "count_at_limit", "count_over_limit"])
def test_narrowed_column_items(lib, case):
    # 2^27 packets over 2^32: the column partition narrows its items to u32 after
    # level 1 when every link count fits; heavy destination buckets are widened back,
    # tiles span several tiny level-1 parents, counts sit at / past the narrow limit
    n = 1 << 27
    rng = np.random.default_rng(31)
    s = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    if case == "hot_dst":
        d[: n // 4] = 0xDEADBEEF
    elif case == "tiny_level1":
        d[: n - n // 100] = rng.integers(0, 1 << 25, n - n // 100, dtype=np.uint64).astype(np.uint32)
    else:
        # a link repeated 2^cb times or once more: 2^27 packets -> D = 18 bits in three
        # 6-bit levels, 26 destination bits below level 1, cb = 32 - 26 = 6
        reps = (1 << 6) + (1 if case == "count_over_limit" else 0)
        s[:reps] = 12345
        d[:reps] = 67890
    assert lib.stats9(s, d, None, 1 << 32) == orc.stats9_packed(s, d)


def test_small_spaces_and_invalid_mix(lib):
    rng = np.random.default_rng(17)
    for _ in range(60):
        n = int(rng.integers(1, 20000))
        space = int(rng.integers(1, 5000))
        s = rng.integers(0, space, n)
        d = rng.integers(0, space, n)
        v = rng.random(n) > 0.3
        assert lib.stats9(s, d, v, space) == orc.stats9_packed(s, d, v)
        w = int(rng.integers(1, n + 1))
        per, _ = orc.stats9_windows_packed(s, d, v, w)
        assert lib.window_stats9(s, d, v, space, w).tolist() == [list(r) for r in per]


def test_heavy_runs_cross_tiles(lib):
    # one link repeated far beyond a 4096-item tile, plus a heavy source / destination
    n = 200_000
    s = np.zeros(n, np.uint32)
    d = np.zeros(n, np.uint32)
    d[100_000:] = np.arange(100_000) % 9000
    s[150_000:] = np.arange(50_000) % 7 + 1
    assert lib.stats9(s, d, None, 1 << 16) == orc.stats9_packed(s, d)


def test_reduce_quirks(lib):
    assert lib.reduce_i64(np.array([1, 2, 3]), lib.REDUCE_SUM) == 6
    assert lib.reduce_i64(np.array([], np.int64), lib.REDUCE_SUM) == 0
    assert lib.reduce_i64(np.array([-5, -2, -9]), lib.REDUCE_MAX) == -2
    big = np.array([2**62, 2**62, 5], dtype=np.int64)
    assert lib.reduce_i64(big, lib.REDUCE_SUM) == int(big.sum())  # int64 wrap
    data = np.random.default_rng(1).integers(-10**12, 10**12, 1_000_003)
    assert lib.reduce_i64(data, lib.REDUCE_SUM) == int(data.sum())
    assert lib.reduce_i64(data, lib.REDUCE_MAX) == int(data.max())


@pytest.mark.parametrize("n", [1000, 1 << 20])
def test_out_of_range_address_rejected_on_device(n):
    """Device columns are range-checked like PacketStream (traffic.py:56-64): an address
    >= address_space raises ValueError (NMX_EINVAL) instead of packing a key wider than
    2b bits (nmx_api.cu stats_device_impl)."""
    import torch

    from paper_2510_14050_b200 import _lib

    space = 1 << 20
    rng = np.random.default_rng(3)
    s = rng.integers(0, space, n).astype(np.uint32)
    d = rng.integers(0, space, n).astype(np.uint32)
    ts = torch.from_numpy(s.view(np.int32)).cuda()
    td = torch.from_numpy(d.view(np.int32)).cuda()
    ok = _lib.stats9(ts, td, None, space)
    assert ok == orc.stats9_packed(s, d)
    td[n // 2] = space  # one address out of range
    with pytest.raises(ValueError, match="address_space"):
        _lib.stats9(ts, td, None, space)
    with pytest.raises(ValueError, match="address_space"):
        _lib.window_stats9(ts, td, None, space, max(1, n // 4))
    d2 = d.copy()
    d2[-1] = 0xFFFFFFFF
    with pytest.raises(ValueError, match="address_space"):
        _lib.stats9(s, d2, None, space)  # host columns (streamed path for large n)
    # the context is still usable afterwards
    td[n // 2] = 0
    assert _lib.stats9(ts, td, None, space)[0] == n


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("lg,space,window", [(16, 1 << 20, 4096), (20, 1 << 24, 1 << 14), (21, 1 << 18, 50_000),
                                             (22, 1 << 26, 1 << 16), (22, (1 << 26) - 3, 65_537),
                                             (23, 1 << 24, 1 << 17)])
def test_windows_msd_path(lib, kind, lg, space, window):
    """Per-window statistics through the windowed MSD path (window id above the
    address bits, b + wb <= 32; power-law inputs with heavy buckets fall back to the
    LSD path) against the packed oracle, window by window, with invalid packets and a
    partial last window."""
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    n = (1 << lg) + 1234
    s, d = gen(23, 0, n, space)
    v = np.random.default_rng(lg).random(n) > 0.1
    s[-5:] = space - 1  # the all-ones source / destination of the last window
    d[-3:] = space - 1
    per, _ = orc.stats9_windows_packed(s, d, v, window)
    assert lib.window_stats9(s, d, v, space, window).tolist() == [list(r) for r in per]
    # device-resident columns, no validity mask
    ds, dd = lib.DeviceArray(n), lib.DeviceArray(n)
    ds.upload(s)
    dd.upload(d)
    per2, _ = orc.stats9_windows_packed(s, d, None, window)
    assert lib.window_stats9(ds, dd, None, space, window).tolist() == [list(r) for r in per2]
    ds.close()
    dd.close()
