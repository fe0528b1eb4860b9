"""Merge-path element-wise addition (K10) and device COO statistics vs the oracle."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def coo():
    from paper_2510_14050_b200 import coo as c

    return c


def _gen(kind, seed, off, n, space):
    g = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    return g(seed, off, n, space)


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("space", [1 << 32, 5000, 7])
def test_coo_from_packets_and_stats(coo, kind, space):
    s, d = _gen(kind, 3, 0, 200_000, space)
    v = np.random.default_rng(1).random(len(s)) > 0.1
    m = coo.coo_from_packets(s, d, v)
    keys, counts = m.download()
    wk, wc = orc.coo_packed(s, d, v)
    assert np.array_equal(keys, wk) and np.array_equal(counts, wc)
    assert m.stats9() == orc.stats9_packed(s, d, v)


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("space", [1 << 32, 3000, 2])
def test_merge_add_equals_concatenation(coo, kind, space):
    s, d = _gen(kind, 5, 0, 300_000, space)
    cut = [0, 70_000, 70_001, 190_000, 300_000]
    parts = [coo.coo_from_packets(s[a:b], d[a:b]) for a, b in zip(cut[:-1], cut[1:])]
    acc = parts[0]
    for p in parts[1:]:
        acc = coo.merge_add(acc, p)
    keys, counts = acc.download()
    wk, wc = orc.coo_packed(s, d)
    assert np.array_equal(keys, wk) and np.array_equal(counts, wc)
    assert acc.stats9() == orc.stats9_packed(s, d)


def test_merge_add_edge_cases(coo):
    e = coo.coo_from_packets(np.zeros(0, np.uint32), np.zeros(0, np.uint32))
    assert e.nnz == 0 and e.stats9() == (0,) * 9
    a = coo.coo_from_packets(np.array([1, 1, 2], np.uint32), np.array([5, 5, 6], np.uint32))
    assert (e + a).download()[1].tolist() == [2, 1]
    assert (a + e).stats9() == a.stats9()
    b = coo.coo_from_packets(np.array([1, 3], np.uint32), np.array([5, 0], np.uint32))
    k, c = (a + b).download()
    assert k.tolist() == [(1 << 32) | 5, (2 << 32) | 6, (3 << 32) | 0] and c.tolist() == [3, 1, 1]
    # identical inputs: every key duplicated across a tile boundary somewhere
    s, d = _gen("uniform", 9, 0, 50_000, 1 << 32)
    x = coo.coo_from_packets(s, d)
    kk, cc = (x + x).download()
    k1, c1 = x.download()
    assert np.array_equal(kk, k1) and np.array_equal(cc, 2 * c1)


def test_streamed_windows_log_structured(coo):
    s, d = _gen("powerlaw", 11, 0, 1 << 20, 1 << 32)
    w = 1 << 16
    got = coo.stream_stats9((s[i:i + w], d[i:i + w]) for i in range(0, len(s), w))
    assert got == orc.stats9_packed(s, d)


def test_streamed_pinned_windows_overlapped(coo):
    from paper_2510_14050_b200 import _lib

    s, d = _gen("uniform", 13, 0, 3 << 18, 1 << 32)
    w = 1 << 18
    wins = []
    for i in range(0, len(s), w):
        ps, pd = _lib.PinnedArray(w), _lib.PinnedArray(w)
        ps.array[:] = s[i:i + w]
        pd.array[:] = d[i:i + w]
        wins.append((ps, pd))
    got = coo.stream_stats9_pinned([(a.array, b.array) for a, b in wins])
    assert got == orc.stats9_packed(s, d)


@pytest.mark.parametrize("overlap", [0.0, 0.5, 1.0])
def test_merge_add_many_tiles(coo, overlap):
    # ~2^20 links per side, a fraction shared (duplicates straddle tile boundaries)
    rng = np.random.default_rng(int(overlap * 10) + 3)
    n = 1 << 20
    s = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    k = int(n * overlap)
    s2 = np.concatenate([s[:k], rng.integers(0, 1 << 32, n - k, dtype=np.uint64).astype(np.uint32)])
    d2 = np.concatenate([d[:k], rng.integers(0, 1 << 32, n - k, dtype=np.uint64).astype(np.uint32)])
    a = coo.coo_from_packets(s, d)
    b = coo.coo_from_packets(s2, d2)
    m = coo.merge_add(a, b)
    keys, counts = m.download()
    wk, wc = orc.coo_packed(np.concatenate([s, s2]), np.concatenate([d, d2]))
    assert np.array_equal(keys, wk) and np.array_equal(counts, wc)
    assert m.stats9() == orc.stats9_packed(np.concatenate([s, s2]), np.concatenate([d, d2]))


@pytest.mark.parametrize("n", [40, 5000])
def test_wide_counts_merge_and_stats(coo, n):
    """u64 counts (the reference's int64 matrix values): merged links beyond 2^32 - 1
    packets keep their exact sums, and the statistics of such a matrix (the 64-bit
    hash-table path) equal the oracle's; a sum beyond 2^63 - 1 is rejected."""
    rng = np.random.default_rng(n)
    src = rng.integers(0, 1 << 32, n, dtype=np.uint64)
    dst = rng.integers(0, 50, n, dtype=np.uint64)  # shared destinations: wide column sums
    keys = np.unique((src << np.uint64(32)) | dst)
    ca = rng.integers(1, 1 << 40, len(keys), dtype=np.int64)
    cb = rng.integers(1, 1 << 40, len(keys), dtype=np.int64)
    a = coo.coo_from_keys(keys, ca)
    b = coo.coo_from_keys(keys[::2], cb[::2])
    k, c = coo.merge_add(a, b).download()
    wk, wc = orc.merge_add_coo(keys, ca, keys[::2], cb[::2])
    assert np.array_equal(k, wk) and np.array_equal(c, wc) and c.max() > (1 << 32)
    assert coo.merge_add(a, b).stats9() == orc.stats9_from_coo(wk, wc)
    big = coo.coo_from_keys(keys[:1], np.array([(1 << 62) + 1], np.int64))
    with pytest.raises(Exception):
        coo.merge_add(big, big)


@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
@pytest.mark.parametrize("lg,space", [(16, 1 << 32), (19, 1 << 20), (21, 1 << 32), (22, (1 << 28) + 5),
                                      (23, 1 << 24)])
def test_coo_sorted_on_msd_path(coo, kind, lg, space):
    """Unique links + counts from the MSD partition and the per-group shared-memory
    sort (power-law heavy buckets take the LSD sort) == the packed oracle, keys in
    order; the same keys through nmx_coo_build (matrix_from_pairs' entry) with a
    tight address space and through windows (build_matrices)."""
    n = (1 << lg) + 777
    s, d = _gen(kind, 41, 0, n, space)
    v = np.random.default_rng(lg).random(n) > 0.05
    m = coo.coo_from_packets(s, d, v)
    keys, counts = m.download()
    wk, wc = orc.coo_packed(s, d, v)
    assert np.array_equal(keys, wk) and np.array_equal(counts, wc)
    assert m.stats9() == orc.stats9_packed(s, d, v)
    m.close()


@pytest.mark.parametrize("space,window", [(1 << 20, 1 << 17), (1 << 16, 100_000), (1 << 24, 1 << 21)])
def test_build_matrices_on_msd_path(space, window):
    from paper_2510_14050_b200 import traffic as nm

    n = (1 << 22) + 99
    s, d = orc.gen_uniform(8, 0, n, space)
    v = np.random.default_rng(3).random(n) > 0.1
    st = nm.PacketStream(src=s.astype(np.int64), dst=d.astype(np.int64), valid=v, address_space=space)
    ours = nm.build_matrices(st, window)
    ref = orc.ref_build_matrices(st.src, st.dst, st.valid, window, space)
    assert len(ours) == len(ref)
    for a, (rp, ci, va) in zip(ours, ref):
        assert np.array_equal(a.row_ptr, rp) and np.array_equal(a.col_idx, ci) and np.array_equal(a.values, va)
