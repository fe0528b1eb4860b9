"""Packet files: the reference's 9-byte record format
(traffic.py:25, write_packets / read_packets traffic.py:370-388).

CPU tests mirror tests/test_traffic.py::TestPacketFiles of the reference and pin
the byte layout; GPU tests check the device path (raw records streamed and
unpacked on the GPU) bit-exactly against the packed-key oracle."""

import struct

import numpy as np
import pytest

from oracle import netmeter_oracle as orc
from paper_2510_14050_b200 import PacketStream, generate_packets, read_packets, write_packets


def test_round_trip(tmp_path):
    stream = generate_packets(1000, 512, seed=6, invalid_fraction=0.1)
    path = tmp_path / "packets.bin"
    write_packets(stream, path)
    back = read_packets(path, address_space=512)
    assert np.array_equal(back.src, stream.src)
    assert np.array_equal(back.dst, stream.dst)
    assert np.array_equal(back.valid, stream.valid)


def test_record_width_is_nine_bytes(tmp_path):
    stream = generate_packets(10, 4, seed=0)
    path = tmp_path / "packets.bin"
    write_packets(stream, path)
    assert path.stat().st_size == 90


def test_byte_layout_little_endian(tmp_path):
    stream = PacketStream(np.array([0x01020304, 7]), np.array([0xA0B0C0D0, 0]), np.array([True, False]), 2**32)
    path = tmp_path / "p.bin"
    write_packets(stream, path)
    assert path.read_bytes() == struct.pack("<IIB", 0x01020304, 0xA0B0C0D0, 1) + struct.pack("<IIB", 7, 0, 0)


def test_address_space_inferred(tmp_path):
    stream = PacketStream(np.array([0, 5]), np.array([2, 1]), np.ones(2, bool), 6)
    path = tmp_path / "p.bin"
    write_packets(stream, path)
    assert read_packets(path).address_space == 6


def test_wide_addresses_rejected(tmp_path):
    stream = PacketStream(np.array([2**32]), np.array([0]), np.ones(1, bool), 2**33)
    with pytest.raises(ValueError):
        write_packets(stream, tmp_path / "p.bin")


def _records(s, d, v):
    r = np.empty(len(s), dtype=np.dtype([("src", "<u4"), ("dst", "<u4"), ("valid", "u1")]))
    r["src"], r["dst"], r["valid"] = s, d, v
    return r


@pytest.mark.gpu
@pytest.mark.parametrize("n,kind", [(5, "uniform"), (7777, "powerlaw"), ((1 << 21) + 3, "uniform"),
                                    ((1 << 22) + 1, "powerlaw")])
def test_stats9_file_matches_oracle(tmp_path, n, kind):
    from paper_2510_14050_b200 import stats9_file

    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = gen(31, 0, n, 1 << 32)
    v = np.random.default_rng(n).random(n) > 0.15
    path = tmp_path / "p.bin"
    _records(s, d, v).tofile(path)
    want = orc.stats9_packed(s, d, v)
    assert stats9_file(path).astuple() == want
    assert stats9_file(path, window_packets=100_003).astuple() == want  # unaligned window starts
    assert stats9_file(path, address_space=1 << 32).astuple() == want


@pytest.mark.gpu
def test_stats9_file_address_range(tmp_path):
    from paper_2510_14050_b200 import stats9_file

    s = np.arange(3000, dtype=np.uint32)
    d = np.full(3000, 5, np.uint32)
    path = tmp_path / "p.bin"
    _records(s, d, np.ones(3000, bool)).tofile(path)
    assert stats9_file(path, address_space=3000).astuple() == orc.stats9_packed(s, d)
    with pytest.raises(ValueError):
        stats9_file(path, address_space=2999)
    big = np.arange(1 << 21, dtype=np.uint32)
    _records(big, big, np.ones(len(big), bool)).tofile(path)
    with pytest.raises(ValueError):
        stats9_file(path, address_space=1 << 20)


@pytest.mark.gpu
def test_unpack_records_device(tmp_path):
    from paper_2510_14050_b200 import _lib

    n = 100_001
    rng = np.random.default_rng(2)
    s = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    d = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    v = rng.random(n) > 0.5
    raw = _records(s, d, v).view(np.uint8)
    dr = _lib.DeviceArray((len(raw) + 3) // 4)
    dr.upload(np.frombuffer(raw.tobytes() + b"\0" * (4 * ((len(raw) + 3) // 4) - len(raw)), np.uint32))
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    dv = _lib.DeviceArray((n + 3) // 4)
    _lib.unpack_records(dr, n, ds, dd, dv)
    assert np.array_equal(ds.download(), s) and np.array_equal(dd.download(), d)
    assert np.array_equal(dv.download().view(np.uint8)[:n] != 0, v)
