"""The reference's hot-path behaviours, re-pointed at the B200 package (SURVEY.md 4
reuse plan): containers, reductions and reports must equal the reference's
(hand vectors from tests/golden/golden.json, the CPU restatement for random
inputs)."""

import threading

import numpy as np
import pytest

import paper_2510_14050_b200 as nm
from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu

HAND = nm.TrafficMatrix(0, 2, [0, 2, 3], [0, 1, 1], [2, 1, 3])
HAND_REPORT = nm.AggregateReport(6, 3, 2, 2, 2, 2)


def test_to_flat_hand_expansion(golden):
    flat = nm.to_flat(HAND)
    for k, want in golden["cases"]["hand"]["flat"].items():
        assert getattr(flat, k).tolist() == want, k


def test_analyze_matrix_hand_and_empty():
    g = nm.make_group_scheduler([2, 2, 2, 2])
    assert nm.analyze_matrix(nm.to_flat(HAND), g, batch_count=2) == HAND_REPORT
    empty = nm.TrafficMatrix(0, 4, [0] * 5, [], [])
    assert nm.analyze_matrix(nm.to_flat(empty), g) == nm.AggregateReport.zero()


def test_reductions():
    g = nm.make_inline_scheduler()
    assert nm.sum_reduce([1, 2, 3], g) == 6
    assert nm.sum_reduce([], g, batch_count=4) == 0
    assert nm.max_scan([3, 7, 2], g) == 7
    assert nm.max_scan([], g, batch_count=3) == 0
    assert nm.max_scan([-5, -2, -9], g, batch_count=2) == -2
    assert nm.max_scan([np.iinfo(np.int64).min], g) == 0
    assert nm.sum_reduce(np.array([2**63 + 5], dtype=np.uint64), g) == -9223372036854775803
    assert nm.sum_reduce(np.array([True, True, False]), g) == 2
    data = np.random.default_rng(21).integers(-1000, 1000, size=100_000)
    assert nm.sum_reduce(data, nm.make_group_scheduler([1] * 8), batch_count=10) == int(data.sum())


@pytest.mark.parametrize("seed", range(6))
def test_matrix_from_pairs_equals_reference_csr(seed):
    rng = np.random.default_rng(seed)
    dim = int(rng.integers(1, 300))
    n = int(rng.integers(0, 5000))
    s, d = rng.integers(0, dim, n), rng.integers(0, dim, n)
    m = nm.matrix_from_pairs(s, d, dim, window_id=seed)
    rp, ci, va = orc.ref_matrix_from_pairs(s, d, dim)
    assert m.window_id == seed and m.dim == dim
    assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci) and np.array_equal(m.values, va)
    flat = nm.to_flat(m)
    ref = orc.ref_to_flat(rp, ci, va, dim)
    for k, v in ref.items():
        assert np.array_equal(getattr(flat, k), v), k


def test_build_matrices_windows():
    s = nm.generate_packets(10, 4, seed=1)
    ms = nm.build_matrices(s, 4)
    assert [int(m.values.sum()) for m in ms] == [4, 4, 2] and [m.window_id for m in ms] == [0, 1, 2]
    s = nm.generate_packets(10_000, 64, seed=77)
    sums = [int(m.values.sum()) for m in nm.build_matrices(s, 512)]
    assert sums == [512] * 19 + [10_000 - 19 * 512]
    st = nm.PacketStream(np.array([0, 0, 1]), np.array([1, 1, 0]), np.array([True, False, True]), 2)
    (m,) = nm.build_matrices(st, 3)
    assert int(m.values.sum()) == 2 and m.to_dense()[0, 1] == 1
    st = nm.PacketStream(np.array([0, 1]), np.array([1, 0]), np.array([False, False]), 2)
    (m,) = nm.build_matrices(st, 8)  # all-invalid window still exists
    assert m.nnz == 0 and nm.analyze_matrix(nm.to_flat(m), nm.make_inline_scheduler()) == nm.AggregateReport.zero()


@pytest.mark.parametrize("space,window", [(64, 100), (4096, 2**12), (300, 7)])
def test_build_matrices_equals_reference(space, window):
    s = nm.generate_packets(20_000, space, seed=space, invalid_fraction=0.1)
    ours = nm.build_matrices(s, window)
    ref = orc.ref_build_matrices(s.src, s.dst, s.valid, window, space)
    assert len(ours) == len(ref)
    for t, (m, (rp, ci, va)) in enumerate(zip(ours, ref)):
        assert m.window_id == t
        assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci) and np.array_equal(m.values, va)


def test_analyze_dataset_and_windows_match_reference(golden):
    c = golden["cases"]["invariance"]
    s = nm.generate_packets(c["n"], c["space"], seed=c["seed"])
    a, _ = nm.anonymize(s, key=c["anon_key"])
    ms = nm.build_matrices(a, c["window"])
    assert len(ms) == 8
    flats = [nm.to_flat(m) for m in ms]
    reference = nm.analyze_dataset(flats, nm.make_inline_scheduler())
    for resources in (1, 2, 4, 8):
        for batches in (1, 5, 10):
            assert nm.analyze_dataset(flats, nm.make_group_scheduler([1] * resources), batches) == reference
    per, tot = reference
    assert [list(orc.to6(w)) for w in c["windows9"]] == [list(r.to_dict().values()) for r in per]
    assert list(tot.to_dict().values()) == c["totals6"]
    wper, wtot = nm.analyze_windows(a, c["window"])
    assert [w.astuple() for w in wper] == [tuple(w) for w in c["windows9"]]
    assert wtot.report() == tot


def test_summed_and_oracle_entry_points(golden):
    c = golden["cases"]["cfg1"]
    s = nm.generate_packets(c["n"], c["space"], seed=c["seed"])
    a, _ = nm.anonymize(s, key=c["anon_key"])
    assert nm.stats9(a).astuple() == tuple(c["stats9"])
    half = len(a) // 2
    parts = [nm.PacketStream(a.src[:half], a.dst[:half], a.valid[:half], a.address_space),
             nm.PacketStream(a.src[half:], a.dst[half:], a.valid[half:], a.address_space)]
    assert nm.analyze_summed(parts).astuple() == tuple(c["stats9"])
    assert nm.oracle_analyze([(0, 1), (0, 1), (1, 0)]) == nm.AggregateReport(3, 2, 2, 1, 2, 1)
    assert nm.oracle_analyze([]) == nm.AggregateReport.zero()


def test_concurrent_analysis_on_one_scheduler():
    rng = np.random.default_rng(91)
    g = nm.make_group_scheduler([2, 2, 2, 2])
    flats, expected = [], []
    for _ in range(8):
        n = int(rng.integers(1, 400))
        s, d = rng.integers(0, 32, n), rng.integers(0, 32, n)
        flats.append(nm.to_flat(nm.matrix_from_pairs(s, d, 32)))
        expected.append(nm.AggregateReport(*orc.to6(orc.oracle_analyze_pairs(zip(s, d)))))
    got = [None] * 8

    def work(k):
        got[k] = nm.analyze_matrix(flats[k], g, 2)

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got == expected


@pytest.mark.parametrize("n,space,kind", [(1000, 7, "uniform"), (70_000, 1 << 20, "powerlaw"),
                                          ((1 << 24) + 12345, 1 << 32, "uniform"), ((1 << 25) + 3, 5000, "powerlaw")])
def test_stats9_of_packet_stream_int64_columns(n, space, kind):
    """analytics.stats9(PacketStream): the stream's own int64 columns through
    nmx_stats9_host_i64 (threaded narrowing into pinned slots, several windows when
    n > 2^24, invalid packets) equal the oracle; out-of-range columns are rejected."""
    import numpy as np

    from oracle import netmeter_oracle as orc
    from paper_2510_14050_b200 import _lib
    from paper_2510_14050_b200.analytics import stats9
    from paper_2510_14050_b200.traffic import PacketStream

    g = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = g(31, 0, n, space)
    v = np.random.default_rng(n).random(n) >= 0.15
    st = PacketStream(src=s.astype(np.int64), dst=d.astype(np.int64), valid=v, address_space=space)
    assert stats9(st).astuple() == orc.stats9_packed(s, d, v)
    bad = s.astype(np.int64)
    bad[n // 2] = space if space < (1 << 32) else -1
    with pytest.raises(ValueError, match="address"):
        _lib.stats9_i64(bad, d.astype(np.int64), v, space)
