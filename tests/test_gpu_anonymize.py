"""GPU anonymize vs the reference restatement
oracle.anonymize (traffic.py:107-137, itself pinned to the reference's own
outputs through the cfg1 / cfg2 / invariance golden cases): identical relabelled
streams, address space and distinct -> code table."""

import numpy as np
import pytest

import paper_2510_14050_b200 as nm
from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


def _oracle_map(src, dst, key):
    inter = np.empty(2 * len(src), np.int64)
    inter[0::2], inter[1::2] = src, dst
    s2, d2, _ = orc.anonymize(src, dst, key)
    out = np.empty(2 * len(src), np.int64)
    out[0::2], out[1::2] = s2, d2
    return dict(zip(inter.tolist(), out.tolist()))


@pytest.mark.parametrize("n,space,seed,key", [(0, 5, 1, 3), (1, 5, 1, 3), (1000, 1, 2, 7), (5000, 77, 42, 9),
                                              (100_000, 2**32, 3, 11), ((1 << 21) + 5, 2**20, 4, 12345)])
def test_anonymize_matches_restatement(n, space, seed, key):
    s = nm.generate_packets(n, space, seed=seed, invalid_fraction=0.1)
    a, amap = nm.anonymize(s, key=key)
    rs, rd, rspace = orc.anonymize(s.src, s.dst, key)
    assert np.array_equal(a.src, rs) and np.array_equal(a.dst, rd) and a.address_space == rspace
    assert np.array_equal(a.valid, s.valid)
    assert amap.key == key and len(amap.mapping) == (rspace if n else 0)
    assert sorted(amap.mapping.values()) == list(range(len(amap.mapping)))
    if n <= 5000:
        assert dict(amap.mapping) == _oracle_map(s.src, s.dst, key)
    if n:
        assert amap.mapping[int(s.src[0])] == int(a.src[0])
    with pytest.raises(KeyError):
        amap.mapping[-1]


def test_anonymize_golden_cfg1(golden):
    c = golden["cases"]["cfg1"]
    s = nm.generate_packets(c["n"], c["space"], seed=c["seed"])
    a, _ = nm.anonymize(s, key=c["anon_key"])
    assert nm.stats9(a).astuple() == tuple(c["stats9"])
    rs, rd, rspace = orc.anonymize(s.src, s.dst, c["anon_key"])
    assert np.array_equal(a.src, rs) and np.array_equal(a.dst, rd) and a.address_space == rspace


def test_anonymize_device_extremes():
    from paper_2510_14050_b200 import _lib

    src = np.array([0xFFFFFFFF, 0, 0xFFFFFFFF, 7, 7], np.uint32)
    dst = np.array([0, 0xFFFFFFFF, 5, 5, 0xFFFFFFFF], np.uint32)
    so, do, k, distinct, code = _lib.anonymize_device(src, dst, 99)
    rs, rd, rspace = orc.anonymize(src.astype(np.int64), dst.astype(np.int64), 99)
    assert k == rspace == 4
    assert np.array_equal(so.download()[:5], rs) and np.array_equal(do.download()[:5], rd)
    assert distinct.tolist() == [0, 5, 7, 0xFFFFFFFF]


def test_wide_addresses_rejected():
    s = nm.PacketStream(np.array([2**32]), np.array([0]), np.ones(1, bool), 2**33)
    with pytest.raises(ValueError):
        nm.anonymize(s, key=1)
