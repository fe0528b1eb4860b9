"""Small calls replayed as one CUDA graph (run_pipeline_msd_graph in nmx_api.cu):
a repeated call on the same device buffers records its launch sequence once and
replays it; every replay must equal the oracle, including after the buffers' contents
change, after other calls moved the library's workspace, when a replay meets a heavy
bucket (discarded, rerun the ordinary way) and when an address is out of range."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


def _dev(a):
    from paper_2510_14050_b200 import _lib

    d = _lib.DeviceArray(len(a))
    d.upload(np.ascontiguousarray(a, dtype=np.uint32))
    return d


@pytest.mark.parametrize("lg,space", [(16, 1 << 32), (17, 1 << 18), (20, 5000), (23, 1 << 24)])
def test_replays_equal_oracle(lg, space):
    from paper_2510_14050_b200 import _lib

    n = 1 << lg
    ctx = _lib.context(0)
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    for seed in (3, 4, 5):  # same buffers, new contents each round
        s, d = orc.gen_uniform(seed, 0, n, space)
        ds.upload(s)
        dd.upload(d)
        want = orc.stats9_packed(s, d)
        for _ in range(3):
            assert _lib.stats9(ds, dd, None, space) == want
        assert len(ctx.last_timing()["stages_ms"]) == 1  # a replay: one graph launch, one interval


def test_replay_after_workspace_moved():
    from paper_2510_14050_b200 import _lib

    n = 1 << 18
    s, d = orc.gen_uniform(9, 0, n, 1 << 32)
    ds, dd = _dev(s), _dev(d)
    want = orc.stats9_packed(s, d)
    assert _lib.stats9(ds, dd, None, 1 << 32) == want
    assert _lib.stats9(ds, dd, None, 1 << 32) == want
    # a larger call grows the context's buffers: the recorded graph must not be replayed
    s2, d2 = orc.gen_uniform(10, 0, 1 << 22, 1 << 32)
    assert _lib.stats9(_dev(s2), _dev(d2), None, 1 << 32) == orc.stats9_packed(s2, d2)
    for _ in range(2):
        assert _lib.stats9(ds, dd, None, 1 << 32) == want


def test_replay_meeting_heavy_buckets_reruns():
    from paper_2510_14050_b200 import _lib

    n = 1 << 18
    s, d = orc.gen_uniform(11, 0, n, 1 << 32)
    ds, dd = _dev(s), _dev(d)
    assert _lib.stats9(ds, dd, None, 1 << 32) == orc.stats9_packed(s, d)
    assert _lib.stats9(ds, dd, None, 1 << 32) == orc.stats9_packed(s, d)  # recorded
    # same buffers, now one source with 5000 packets (a heavy bucket the graph lacks)
    s[:5000] = 77
    ds.upload(s)
    for _ in range(2):
        assert _lib.stats9(ds, dd, None, 1 << 32) == orc.stats9_packed(s, d)


def test_replay_rejects_out_of_range_addresses():
    from paper_2510_14050_b200 import _lib

    n, space = 1 << 17, 1 << 20
    s, d = orc.gen_uniform(12, 0, n, space)
    ds, dd = _dev(s), _dev(d)
    want = orc.stats9_packed(s, d)
    assert _lib.stats9(ds, dd, None, space) == want
    assert _lib.stats9(ds, dd, None, space) == want
    bad = d.copy()
    bad[123] = space + 5
    dd.upload(bad)
    with pytest.raises(ValueError, match="address"):
        _lib.stats9(ds, dd, None, space)
    dd.upload(d)
    assert _lib.stats9(ds, dd, None, space) == want


def test_valid_flags_and_power_law_replays():
    from paper_2510_14050_b200 import _lib

    n = 1 << 20
    s, d = orc.gen_powerlaw(13, 0, n, 1 << 32)
    v = (np.random.default_rng(2).random(n) >= 0.25).astype(np.uint8)
    ds, dd, dv = _dev(s), _dev(d), _lib.DeviceArray(n, itemsize=1)
    dv.upload(v)
    want = orc.stats9_packed(s, d, v.astype(bool))
    for _ in range(3):
        assert _lib.stats9(ds, dd, dv, 1 << 32) == want


@pytest.mark.parametrize("lg,space,window", [(20, 1 << 20, 1 << 14), (23, 1 << 24, 1 << 17), (22, 5000, 100_000)])
def test_window_replays_equal_oracle(lg, space, window):
    """Per-window statistics on the MSD path recorded as one graph: replays on the same
    buffers with new contents, a replay meeting heavy buckets (power-law: rerun on the
    LSD path), and a replay seeing an out-of-range address."""
    from paper_2510_14050_b200 import _lib

    n = (1 << lg) + 5
    ctx = _lib.context(0)
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    for seed, gen in ((3, orc.gen_uniform), (4, orc.gen_uniform), (5, orc.gen_powerlaw), (6, orc.gen_uniform)):
        s, d = gen(seed, 0, n, space)
        ds.upload(s)
        dd.upload(d)
        per, _ = orc.stats9_windows_packed(s, d, None, window)
        want = [list(r) for r in per]
        for _ in range(3):
            assert _lib.window_stats9(ds, dd, None, space, window).tolist() == want
    if gen is orc.gen_uniform and space < (1 << 32):
        bad = d.copy()
        bad[n // 3] = space
        dd.upload(bad)
        with pytest.raises(ValueError, match="address_space"):
            _lib.window_stats9(ds, dd, None, space, window)
    assert ctx is not None
