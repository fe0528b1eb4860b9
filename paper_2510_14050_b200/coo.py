"""Device-resident traffic matrices (sorted unique COO) and their element-wise sum.

SURVEY.md 8(a) a11: the summed matrix A = sum_t A_t of several windows is the
count matrix of the concatenated valid packets (build_matrices(stream,
window_size=len(stream)), traffic.py:221-242). Here each window becomes a
``DeviceCOO`` (``nmx_coo_from_packets``) and windows are combined with the
merge-path kernel (``nmx_coo_merge_add``) -- the streaming form used when the
packets do not fit the device at once (BASELINE config 5). Keys are
(src << 32) | dst, counts u64 (int64 on the host).
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable

import numpy as np

from . import _lib


class DeviceCOO:
    """Sorted unique (key, count) links on one GPU; freed with ``close()`` / GC."""

    def __init__(self, handle: C.c_void_p, device: int = 0):
        self._h = handle
        self.device = device
        self._ctx = _lib.context(device)

    @property
    def nnz(self) -> int:
        n = C.c_uint64()
        _lib.check(self._ctx._lib.nmx_coo_nnz(self._h, C.byref(n)))
        return n.value

    def stats9(self) -> tuple:
        out = np.zeros(9, dtype=np.int64)
        _lib.check(self._ctx._lib.nmx_coo_stats9(self._ctx.handle, self._h, out.ctypes.data))
        return tuple(int(x) for x in out)

    def download(self):
        """(keys uint64 (src<<32)|dst, counts int64) on the host."""
        n = self.nnz
        keys = np.empty(n, dtype=np.uint64)
        counts = np.empty(n, dtype=np.int64)
        _lib.check(self._ctx._lib.nmx_coo_download(self._ctx.handle, self._h, keys.ctypes.data, counts.ctypes.data))
        return keys, counts

    def __add__(self, other: "DeviceCOO") -> "DeviceCOO":
        return merge_add(self, other)

    def close(self) -> None:
        if self._h:
            self._ctx._lib.nmx_coo_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def reserve(nbytes: int, device: int = 0) -> None:
    """Keep ``nbytes`` of device memory mapped in the COO allocation pool."""
    ctx = _lib.context(device)
    _lib.check(ctx._lib.nmx_coo_reserve(ctx.handle, int(nbytes)))


def coo_from_packets(src, dst, valid=None, device: int = 0) -> DeviceCOO:
    """Unique links of one window. ``src``/``dst``: host arrays (copied) or device arrays."""
    ctx = _lib.context(device)
    keep = []
    if not _lib._is_device(src):
        s = _lib._u32_host(src)
        d = _lib._u32_host(dst)
        n = len(s)
        ds, dd = _lib.DeviceArray(n, device=device), _lib.DeviceArray(n, device=device)
        if n:
            ds.upload(s)
            dd.upload(d)
        dv = None
        if valid is not None:
            v = _lib._valid_host(valid)
            dv = _lib.DeviceArray(n, itemsize=1, device=device)
            if n:
                dv.upload(v)
        keep = [ds, dd, dv]
        src, dst, valid = ds, dd, dv
    n = int(src.numel())
    h = C.c_void_p()
    _lib.check(ctx._lib.nmx_coo_from_packets(ctx.handle, _lib._ptr(src), _lib._ptr(dst), _lib._ptr(valid), n,
                                             C.byref(h)))
    del keep
    return DeviceCOO(h, device)


def coo_from_keys(keys, counts, device: int = 0) -> DeviceCOO:
    """Upload host sorted unique keys ((src << 32) | dst) with counts as a DeviceCOO."""
    ctx = _lib.context(device)
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    c = np.ascontiguousarray(counts, dtype=np.int64)
    if len(k) != len(c):
        raise ValueError("keys and counts must have equal lengths")
    h = C.c_void_p()
    _lib.check(ctx._lib.nmx_coo_upload(ctx.handle, k.ctypes.data, c.ctypes.data, len(k), C.byref(h)))
    return DeviceCOO(h, device)


def merge_add(a: DeviceCOO, b: DeviceCOO) -> DeviceCOO:
    """Element-wise sum C = A + B (merge path over sorted keys)."""
    ctx = _lib.context(a.device)
    h = C.c_void_p()
    _lib.check(ctx._lib.nmx_coo_merge_add(ctx.handle, a._h, b._h, C.byref(h)))
    return DeviceCOO(h, a.device)


class SummedMatrix:
    """Running sum of window matrices with log-structured merging: runs of equal
    rank are merged pairwise (like a binary counter), so every link is merged
    O(log windows) times instead of once per window."""

    def __init__(self, device: int = 0):
        self.device = device
        self._runs: list[tuple[int, DeviceCOO]] = []  # (rank, coo), ranks strictly decreasing

    def add(self, coo: DeviceCOO) -> None:
        rank = 0
        while self._runs and self._runs[-1][0] == rank:
            _, prev = self._runs.pop()
            merged = merge_add(prev, coo)
            prev.close()
            coo.close()
            coo, rank = merged, rank + 1
        self._runs.append((rank, coo))

    def result(self) -> DeviceCOO:
        if not self._runs:
            return coo_from_packets(np.zeros(0, np.uint32), np.zeros(0, np.uint32), device=self.device)
        acc = self._runs.pop()[1]
        while self._runs:
            _, prev = self._runs.pop()
            merged = merge_add(prev, acc)
            prev.close()
            acc.close()
            acc = merged
        self._runs = [(99, acc)]
        return acc


def stream_stats9(windows: Iterable, device: int = 0) -> tuple:
    """Nine statistics of the matrix summed over a stream of packet windows
    ((src, dst) or (src, dst, valid) host or device arrays per window)."""
    acc = SummedMatrix(device)
    for w in windows:
        acc.add(coo_from_packets(*w, device=device))
    return acc.result().stats9()


def stream_stats9_pinned(windows, device: int = 0, address_space: int = 1 << 32) -> tuple:
    """BASELINE config 5: windows of packets in (pinned) host memory streamed to the
    device (nmx_stream_stats9): the H2D copy of window t+1 runs on a second stream
    while window t is partitioned into the device-resident running sum; the
    remaining partition levels and the statistics run once over the sum.
    ``windows``: list of (src, dst[, valid]) host arrays."""
    return _lib.stream_stats9(windows, address_space, device)
