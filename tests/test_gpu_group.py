"""Device groups (nmx_group_*, resources.DeviceGroup): G ranks driven by one process,
the sharded owner(src) / owner(dst) pipeline with in-library peer-copy exchanges.
On a one-GPU box the ranks are virtual (all on cuda:0, each with its own context and
stream); the same code path runs G distinct B200s over NVLink."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


def _packets(kind, n, space, seed, invalid=0.0):
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = gen(seed, 0, n, space)
    v = None
    if invalid:
        v = np.random.default_rng(seed).random(n) >= invalid
    return s, d, v


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_group_host_matches_oracle(G, kind):
    from paper_2510_14050_b200 import _lib

    s, d, v = _packets(kind, 1 << 20, 1 << 32, 5, invalid=0.1)
    want = orc.stats9_packed(s, d, v)
    grp = _lib.Group([0] * G)
    try:
        for b in (1, 5):
            assert grp.stats9_host(s, d, v, 1 << 32, batch_count=b) == want
        x1, x2 = grp.last_exchange()
        assert x1 == 8 * want[0]  # every valid packet crosses exchange 1 once
        assert x2 == 8 * want[1]  # every unique link's (dst, count) crosses exchange 2 once
    finally:
        grp.close()


@pytest.mark.parametrize("G", [2, 8])
@pytest.mark.parametrize("lg,space", [(24, 1 << 32), (22, 1 << 16), (12, 300), (5, 7)])
def test_group_sizes_and_spaces(G, lg, space):
    from paper_2510_14050_b200 import _lib

    s, d, _ = _packets("powerlaw", 1 << lg, space, 9)
    grp = _lib.Group([0] * G)
    try:
        assert grp.stats9_host(s, d, None, space) == orc.stats9_packed(s, d)
    finally:
        grp.close()


def test_group_device_columns_and_empty_ranks():
    from paper_2510_14050_b200 import _lib

    G = 4
    n = 1 << 18
    s, d, _ = _packets("uniform", n, 1 << 20, 3)
    lens = [n // 2, 0, n // 2 - 1000, 1000]  # one rank holds nothing
    grp = _lib.Group([0] * G)
    arrs = []
    try:
        at = 0
        srcs, dsts = [], []
        for ln in lens:
            a, b = _lib.DeviceArray(ln), _lib.DeviceArray(ln)
            if ln:
                a.upload(s[at:at + ln])
                b.upload(d[at:at + ln])
            at += ln
            srcs.append(a)
            dsts.append(b)
            arrs += [a, b]
        assert grp.stats9_device(srcs, dsts, 1 << 20) == orc.stats9_packed(s, d)
    finally:
        for a in arrs:
            a.close()
        grp.close()


def test_group_error_propagates_and_recovers():
    from paper_2510_14050_b200 import _lib

    s, d, _ = _packets("uniform", 1 << 16, 1 << 12, 4)
    bad = d.copy()
    bad[-7] = 1 << 12  # out of range, lands on the last rank's span
    grp = _lib.Group([0] * 3)
    try:
        with pytest.raises(ValueError, match="address_space"):
            grp.stats9_host(s, bad, None, 1 << 12)
        assert grp.stats9_host(s, d, None, 1 << 12) == orc.stats9_packed(s, d)
    finally:
        grp.close()


def test_dropin_scheduler_dispatch(golden):
    """The reference API with make_group_scheduler(G): stats9 / analyze_summed shard the
    stream, analyze_windows / analyze_dataset spread windows, sum_reduce / max_scan
    spread the view -- all equal to the reference's own outputs."""
    import paper_2510_14050_b200 as nm

    c = golden["cases"]["windows_invalid"]
    st = nm.generate_packets(c["n"], c["space"], c["seed"], invalid_fraction=c["invalid_fraction"])
    for G in (1, 2, 4, 8):
        with nm.make_group_scheduler(G) as g:
            for b in (1, 5, 10):
                assert nm.stats9(st, scheduler=g, batch_count=b).astuple() == tuple(c["stats9"])
            per, tot = nm.analyze_windows(st, c["window"], scheduler=g)
            assert [list(r.astuple()) for r in per] == c["windows9"]
            mats = nm.build_matrices(st, c["window"])
            reps, tot6 = nm.analyze_dataset(mats, g, batch_count=3)
            assert [list(orc.to6(w)) for w in c["windows9"]] == [
                [r.valid_packets, r.unique_links, r.unique_sources, r.max_fanout, r.unique_destinations, r.max_fanin]
                for r in reps]
            assert orc.to6(tot.astuple()) == tuple(c["totals6"])
            data = np.random.default_rng(G).integers(-2**62, 2**62, 100_003)
            assert nm.sum_reduce(data, g, batch_count=7) == int(np.add.reduce(data))
            assert nm.max_scan(data, g, batch_count=7) == int(data.max())
            assert nm.max_scan([], g, batch_count=3) == 0


def test_group_uses_every_rank_context():
    """analyze_dataset over a group really runs on the ranks' own contexts."""
    import threading

    import paper_2510_14050_b200 as nm
    from paper_2510_14050_b200 import _lib

    seen = set()
    real = _lib.reduce_i64
    lock = threading.Lock()

    def spy(a, op, device=0):
        with lock:
            seen.add(_lib.context(device).handle.value)
        return real(a, op, device)

    rng = np.random.default_rng(1)
    mats = [nm.matrix_from_pairs(rng.integers(0, 50, 500), rng.integers(0, 50, 500), 50, window_id=k)
            for k in range(8)]
    _lib.reduce_i64 = spy
    try:
        with nm.make_group_scheduler(4) as g:
            nm.analyze_dataset(mats, g)
            handles = {c.handle.value for c in g.native.contexts}
    finally:
        _lib.reduce_i64 = real
    assert handles <= seen and len(handles) == 4
