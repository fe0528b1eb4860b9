"""The CPU oracle (oracle/netmeter_oracle.py) pinned against the reference's
own outputs recorded in tests/golden/golden.json (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc


def _pairs(case):
    p = np.array(case["pairs"], dtype=np.int64).reshape(-1, 2)
    valid = np.array(case.get("valid", [1] * len(p)), dtype=bool)
    return p[:, 0], p[:, 1], valid


@pytest.mark.parametrize("name", ["hand", "hand_other", "oracle_hand", "self_loops", "invalid_hand"])
def test_hand_vectors(golden, name):
    case = golden["cases"][name]
    s, d, v = _pairs(case)
    dim = int(max(s.max(), d.max())) + 1
    assert orc.ref_stats9(s, d, v, dim) == tuple(case["stats9"])
    assert orc.stats9_packed(s, d, v) == tuple(case["stats9"])
    assert orc.oracle_analyze_pairs(zip(s[v], d[v])) == tuple(case["stats9"])


def test_hand_flat(golden):
    case = golden["cases"]["hand"]
    s, d, v = _pairs(case)
    flat = orc.ref_to_flat(*orc.ref_matrix_from_pairs(s, d, 2), 2)
    for k, want in case["flat"].items():
        assert flat[k].tolist() == want, k


def test_corpus(golden):
    for c in golden["cases"]["corpus"]:
        s, d, v = orc.generate_packets(c["n"], c["space"], c["seed"], c["invalid_fraction"])
        want = tuple(c["stats9"])
        assert orc.stats9_packed(s, d, v) == want
        if c["n"] <= 3000:
            assert orc.ref_stats9(s, d, v, c["space"]) == want
            assert orc.oracle_analyze_pairs(zip(s[v], d[v])) == want


@pytest.mark.parametrize("name", ["cfg1", "windows_small", "windows_invalid", "invariance"])
def test_generate_anonymize_cases(golden, name):
    c = golden["cases"][name]
    s, d, v = orc.generate_packets(c["n"], c["space"], c["seed"], c["invalid_fraction"])
    space = c["space"]
    if c["anon_key"] is not None:
        s, d, space = orc.anonymize(s, d, c["anon_key"])
    assert space == c["address_space"]
    assert orc.checksum_u32(s) == c["src_sha"] and orc.checksum_u32(d) == c["dst_sha"]
    assert orc.stats9_packed(s, d, v) == tuple(c["stats9"])
    if "window" in c:
        per, tot = orc.stats9_windows_packed(s, d, v, c["window"])
        assert [list(r) for r in per] == c["windows9"]
        assert orc.to6(tot) == tuple(c["totals6"])
        ref_per, ref_tot = orc.ref_analyze_dataset(s, d, v, c["window"], space)
        assert [list(r) for r in ref_per] == c["windows9"]


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_splitmix_cases(golden, kind):
    for name, c in golden["cases"]["splitmix"].items():
        if c["kind"] != kind or c["n"] > 2**22:
            continue
        gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
        s, d = gen(c["seed"], 0, c["n"], c["space"])
        assert orc.checksum_u32(s) == c["src_sha"] and orc.checksum_u32(d) == c["dst_sha"], name
        assert orc.stats9_packed(s, d) == tuple(c["stats9"]), name


def test_generator_chunk_addressable():
    s, d = orc.gen_uniform(3, 0, 1000)
    s2, d2 = orc.gen_uniform(3, 400, 600)
    assert np.array_equal(s[400:], s2) and np.array_equal(d[400:], d2)
    s, d = orc.gen_powerlaw(3, 0, 1000, 1000)
    assert s.max() < 1000 and d.max() < 1000


def test_merge_add_equals_concatenation():
    rng = np.random.default_rng(5)
    s = rng.integers(0, 50, 3000)
    d = rng.integers(0, 50, 3000)
    ka, ca = orc.coo_packed(s[:1700], d[:1700])
    kb, cb = orc.coo_packed(s[1700:], d[1700:])
    k, c = orc.merge_add_coo(ka, ca, kb, cb)
    kw, cw = orc.coo_packed(s, d)
    assert np.array_equal(k, kw) and np.array_equal(c, cw)
    assert orc.stats9_from_coo(k, c) == orc.stats9_packed(s, d)


def test_max_scan_quirks():
    assert orc._max0([]) == 0
    assert orc._max0([np.iinfo(np.int64).min]) == 0
    assert orc._max0([-5, -2, -9]) == -2


# ---------------------------------------------------------------------------
# the bounded-RAM chunked oracle (oracle/nmx_oracle.c) behind tests/golden/full_size.json
# ---------------------------------------------------------------------------
def test_chunked_oracle_pinned_to_reference_goldens(golden):
    from oracle import big

    for name, c in golden["cases"]["splitmix"].items():
        if c["n"] > 1 << 22:
            continue
        kind = big.UNIFORM if c["kind"] == "uniform" else big.POWERLAW
        for bb in (0, 3):  # one bucket, and 8 buckets (the chunked path)
            assert big.stats9_gen(kind, c["seed"], 0, c["n"], c["space"], bucket_bits=bb) == tuple(c["stats9"]), name


def test_chunked_oracle_generator_equals_numpy():
    from oracle import big

    for kind, gen in ((big.UNIFORM, orc.gen_uniform), (big.POWERLAW, orc.gen_powerlaw)):
        for space in (1 << 32, 1 << 20, 300):
            s, d = big.generate(kind, 11, 12345, 4096, space)
            s2, d2 = gen(11, 12345, 4096, space)
            assert np.array_equal(s, s2) and np.array_equal(d, d2)


@pytest.mark.parametrize("seed", [1, 2])
def test_chunked_oracle_pairs_with_invalid(seed):
    from oracle import big

    rng = np.random.default_rng(seed)
    n = 20000
    hot = rng.integers(0, 1 << 32, 8, dtype=np.uint64).astype(np.uint32)
    s = np.where(rng.random(n) < 0.3, hot[rng.integers(0, 8, n)], rng.integers(0, 1 << 32, n, dtype=np.uint64))
    d = np.where(rng.random(n) < 0.3, hot[rng.integers(0, 8, n)], rng.integers(0, 1 << 32, n, dtype=np.uint64))
    s, d = s.astype(np.uint32), d.astype(np.uint32)
    v = rng.random(n) < 0.8
    for bb in (0, 4, 9):
        assert big.stats9_pairs(s, d, v, bucket_bits=bb) == orc.stats9_packed(s, d, v)
    assert big.stats9_pairs(s[:0], d[:0]) == (0,) * 9


def test_full_size_goldens_recorded():
    """tests/golden/full_size.json (oracle/make_full_size.py) holds the BASELINE-size cases."""
    import json
    from pathlib import Path

    p = Path(__file__).resolve().parent / "golden" / "full_size.json"
    g = json.loads(p.read_text())
    for name in ("cfg3_seed7", "cfg3_seed11", "cfg4_seed7", "cfg4_seed11"):
        c = g["cases"][name]
        assert c["n"] == 1 << 30 and c["stats9"][0] == 1 << 30
    assert any(r.startswith("uniform_2^24") for r in g["pinned_against"]["reference_goldens"])
