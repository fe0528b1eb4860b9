"""GPU parity of nmx_stats9_host_batches: a run of independent host batches whose
H2D copies overlap the previous batch's device work. Each batch's nine statistics
must equal the packed-key oracle of that batch alone (and nmx_stats9_host of it),
whatever the neighbouring batches hold: empty batches, invalid packets, sizes on
both sides of the graph / MSD thresholds, power-law heavy buckets, narrow address
spaces, and a bad address in the middle of the run."""

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2510_14050_b200 import _lib

    _lib.context(0)
    return _lib


def test_mixed_batches_equal_oracle(lib):
    rng = np.random.default_rng(5)
    batches, want = [], []
    for i, (gen, n) in enumerate([(orc.gen_uniform, 1 << 20), (orc.gen_powerlaw, 1 << 22), (orc.gen_uniform, 0),
                                  (orc.gen_uniform, 1000), (orc.gen_powerlaw, (1 << 21) + 17),
                                  (orc.gen_uniform, 1 << 22), (orc.gen_uniform, 1 << 16)]):
        s, d = gen(100 + i, 0, n, 1 << 32)
        if i % 2:
            v = rng.random(n) > 0.25
            batches.append((s, d, v))
            want.append(orc.stats9_packed(s, d, v))
        else:
            batches.append((s, d))
            want.append(orc.stats9_packed(s, d))
    got = lib.stats9_batches(batches, 1 << 32)
    assert got == want
    # the same batch through the single-call entry
    assert lib.stats9(*batches[1]) == want[1]


def test_repeated_pinned_batch(lib):
    n = 1 << 23
    s, d = orc.gen_uniform(7, 0, n, 1 << 32)
    hs, hd = lib.PinnedArray(n), lib.PinnedArray(n)
    hs.array[:] = s
    hd.array[:] = d
    want = orc.stats9_packed(s, d)
    assert lib.stats9_batches([(hs.array, hd.array)] * 5, 1 << 32) == [want] * 5
    hs.close()
    hd.close()


def test_narrow_space_and_bad_address(lib):
    space = 1 << 20
    s1, d1 = orc.gen_uniform(3, 0, 1 << 18, space)
    s2, d2 = orc.gen_uniform(4, 0, 1 << 19, space)
    assert lib.stats9_batches([(s1, d1), (s2, d2)], space) == [orc.stats9_packed(s1, d1), orc.stats9_packed(s2, d2)]
    bad = d2.copy()
    bad[12345] = space  # outside [0, address_space)
    with pytest.raises(ValueError):
        lib.stats9_batches([(s1, d1), (s2, bad), (s1, d1)], space)
    # the context stays usable after the failed run
    assert lib.stats9_batches([(s1, d1)], space) == [orc.stats9_packed(s1, d1)]


def test_empty_run(lib):
    assert lib.stats9_batches([], 1 << 32) == []
