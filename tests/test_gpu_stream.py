"""GPU parity of the streamed path (nmx_stream_stats9, BASELINE config 5): host
windows copied on a second stream, level-1 partitioned into one device-resident
running sum; statistics of the summed matrix == the packed-key oracle over the
concatenated valid packets. Also the chunked H2D of
nmx_stats9_host, which uses the same path."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_uneven_windows_with_invalid(lib, kind):
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    rng = np.random.default_rng(11)
    s, d = gen(21, 0, 3 << 20, 1 << 32)
    v = rng.random(len(s)) > 0.2
    cuts = [0, 1000, 1000, 700_000, 2_000_000, 2_000_017, len(s)]
    wins = []
    for i, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        wins.append((s[a:b], d[a:b], v[a:b]) if i % 2 else (s[a:b], d[a:b]))
    vv = np.concatenate([v[a:b] if i % 2 else np.ones(b - a, bool) for i, (a, b) in enumerate(zip(cuts[:-1], cuts[1:]))])
    assert lib.stream_stats9(wins, 1 << 32) == orc.stats9_packed(s, d, vv)


def test_many_windows_pinned(lib):
    w = 1 << 18
    wins, ss, dd = [], [], []
    for k in range(12):
        s, d = orc.gen_powerlaw(3, k * w, w, 1 << 32)
        ps, pd = lib.PinnedArray(w), lib.PinnedArray(w)
        ps.array[:] = s
        pd.array[:] = d
        wins.append((ps, pd))
        ss.append(s)
        dd.append(d)
    got = lib.stream_stats9([(a.array, b.array) for a, b in wins], 1 << 32)
    assert got == orc.stats9_packed(np.concatenate(ss), np.concatenate(dd))
    # repeated windows: the sum doubles every count
    got2 = lib.stream_stats9([(a.array, b.array) for a, b in wins] * 2, 1 << 32)
    assert got2 == orc.stats9_packed(np.concatenate(ss * 2), np.concatenate(dd * 2))


def test_small_and_narrow_spaces_fall_back(lib):
    s, d = orc.gen_uniform(4, 0, 5000, 300)
    assert lib.stream_stats9([(s[:100], d[:100]), (s[100:], d[100:])], 300) == orc.stats9_packed(s, d)
    s, d = orc.gen_uniform(4, 0, 1 << 21, 1 << 8)  # b = 8 < D: single-call LSD path
    assert lib.stream_stats9([(s[: 1 << 20], d[: 1 << 20]), (s[1 << 20 :], d[1 << 20 :])], 1 << 8) == orc.stats9_packed(s, d)
    assert lib.stream_stats9([], 1 << 32) == (0,) * 9
    e = np.zeros(0, np.uint32)
    assert lib.stream_stats9([(e, e), (e, e)], 1 << 32) == (0,) * 9


def test_all_invalid_stream(lib):
    s, d = orc.gen_uniform(5, 0, 1 << 21, 1 << 32)
    v = np.zeros(len(s), bool)
    assert lib.stream_stats9([(s, d, v)], 1 << 32) == (0,) * 9


def test_host_chunked_equals_device(lib):
    s, d = orc.gen_powerlaw(8, 0, (1 << 26) + 12345, 1 << 32)
    got_host = lib.stats9(s, d, None, 1 << 32)
    ds, dd = lib.DeviceArray(len(s)), lib.DeviceArray(len(s))
    ds.upload(s)
    dd.upload(d)
    assert lib.stats9(ds, dd, None, 1 << 32) == got_host


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("space", [1 << 32, 1 << 20])
def test_out_of_core_parts_path(lib, kind, space, monkeypatch):
    """The > 2^31-packet path (source-part arenas, rows per part, destination-part
    arenas, columns per part) forced at small sizes with NMX_PARTS_MIN: equal to the
    one-pass oracle, with invalid packets, uneven windows and records."""
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = gen(31, 0, 5 << 20, space)
    v = np.random.default_rng(5).random(len(s)) > 0.1
    cuts = [0, 3, 1 << 20, 3 << 20, len(s)]
    wins = [(s[a:b], d[a:b], v[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    want = orc.stats9_packed(s, d, v)
    monkeypatch.setenv("NMX_PARTS_MIN", str(1 << 20))
    assert lib.stream_stats9(wins, space) == want
    assert lib.stats9(s, d, v, space) == want  # host entry (2^25-packet chunks) through the same path
    rec = np.zeros(len(s), dtype=np.dtype([("src", "<u4"), ("dst", "<u4"), ("valid", "u1")]))
    rec["src"], rec["dst"], rec["valid"] = s, d, v
    assert lib.stream_records([rec[:1 << 21], rec[1 << 21:]], space) == want
    bad = d.copy()
    if space < 1 << 32:
        bad[-1] = space
        with pytest.raises(ValueError, match="address_space"):
            lib.stream_stats9([(s, bad)], space)


@pytest.mark.parametrize("lg,name", [(31, "cfg5_2^31_seed7"), (32, "cfg5_2^32_seed7")])
def test_cfg5_full_size_golden(lib, lg, name):
    """BASELINE config 5 on one B200: 2^31 / 2^32 packets streamed from pinned host
    memory in 2^28-packet windows (2^32 takes the out-of-core part split), bit-exact
    against the chunked CPU oracle (tests/golden/full_size.json)."""
    import json
    from pathlib import Path

    want = tuple(json.loads((Path(__file__).resolve().parent / "golden" / "full_size.json").read_text())
                 ["cases"][name]["stats9"])
    w = 1 << 28
    ds, dd = lib.DeviceArray(w), lib.DeviceArray(w)
    wins = []
    try:
        for k in range((1 << lg) // w):
            lib.generate(lib.GEN_UNIFORM, 7, k * w, w, 1 << 32, ds, dd)
            ps, pd = lib.PinnedArray(w), lib.PinnedArray(w)
            ps.array[:] = ds.download()
            pd.array[:] = dd.download()
            wins.append((ps, pd))
        ds.close()
        dd.close()
        assert lib.stream_stats9([(a.array, b.array) for a, b in wins], 1 << 32) == want
    finally:
        for a, b in wins:
            a.close()
            b.close()
