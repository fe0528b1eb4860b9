"""Aggregate traffic measures on the B200 (mirrors netmeter.analytics, analytics.py:1-157).

Reference-compatible entry points (same names, argument meaning and errors):
``sum_reduce``, ``max_scan``, ``analyze_matrix``, ``analyze_dataset``,
``oracle_analyze``, ``AggregateReport``. Their reductions run in libnmx.so
(``nmx_reduce_i64``); a device-group scheduler (resources.py) spreads views and
windows over its ranks, and ``batch_count`` chunks each rank's share, as the
reference's resources / batches do.

The hot path (BASELINE.json north star) is ``stats9`` / ``analyze_summed``:
packets -> summed traffic matrix -> the nine Graph Challenge statistics, with
no host-side containers at all (``nmx_stats9_*``), and ``analyze_windows`` for
the per-window (analyze_dataset) semantics (``nmx_window_stats9_*``).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .partitioning import even_spans
from .traffic import FlatContainers, PacketStream, TrafficMatrix, to_flat

_INT64_MIN = np.iinfo(np.int64).min


@dataclass(frozen=True)
class AggregateReport:
    """The six aggregate measures (analytics.py:31-51); key order pinned by the reference tests."""

    valid_packets: int
    unique_links: int
    unique_sources: int
    max_fanout: int
    unique_destinations: int
    max_fanin: int

    def to_dict(self) -> dict[str, int]:
        return asdict(self)

    @classmethod
    def from_dict(cls, data: dict[str, int]) -> "AggregateReport":
        return cls(**{f: int(data[f]) for f in cls.__dataclass_fields__})

    @classmethod
    def zero(cls) -> "AggregateReport":
        return cls(0, 0, 0, 0, 0, 0)


@dataclass(frozen=True)
class Stats9:
    """The nine Graph Challenge statistics of one traffic matrix."""

    valid_packets: int
    unique_links: int
    max_link_packets: int
    unique_sources: int
    max_source_packets: int
    max_fanout: int
    unique_destinations: int
    max_destination_packets: int
    max_fanin: int

    def to_dict(self) -> dict[str, int]:
        return asdict(self)

    def astuple(self) -> tuple:
        return tuple(getattr(self, f) for f in self.__dataclass_fields__)

    def report(self) -> AggregateReport:
        return AggregateReport(self.valid_packets, self.unique_links, self.unique_sources, self.max_fanout,
                               self.unique_destinations, self.max_fanin)

    @classmethod
    def zero(cls) -> "Stats9":
        return cls(0, 0, 0, 0, 0, 0, 0, 0, 0)


def _check_view(data, batch_count: int) -> np.ndarray:
    """analytics.py:68-75 argument rules."""
    if batch_count < 1:
        raise ValueError("batch_count must be >= 1")
    data = np.asarray(data)
    if data.size and data.dtype.kind not in "iub":
        raise TypeError(f"expected an integer view, got dtype {data.dtype}")
    return np.ascontiguousarray(data, dtype=np.int64).reshape(-1)


def _device_of(scheduler) -> int:
    return int(getattr(scheduler, "device", 0) or 0)


def _group(scheduler):
    """The scheduler as a DeviceGroup (None for an unknown SchedulerLike)."""
    from .resources import DeviceGroup

    return scheduler if isinstance(scheduler, DeviceGroup) else None


def _reduce(a: np.ndarray, scheduler, batch_count: int, op: int) -> int:
    """Per-resource partials like the reference's _batched_reduce (analytics.py:54-81):
    the view split by partition_even over the group's ranks, each rank's span in
    batch_count chunks reduced on its own device context, partials combined here
    (SUM wraps mod 2^64 as int64; MAX keeps the INT64_MIN empty sentinel)."""
    g = _group(scheduler)
    if g is None or (g.resource_count == 1 and batch_count == 1) or a.size < 2:
        if g is not None:
            with _lib.using(g.native.contexts[0]):
                return _lib.reduce_i64(a, op)
        return _lib.reduce_i64(a, op, device=_device_of(scheduler))

    def rank_part(r, lo, hi):
        return [_lib.reduce_i64(a[o:o + ln], op) for o, ln in even_spans(lo, hi - lo, batch_count) if ln]

    parts = [v for chunk in g.map_ranks(len(a), rank_part) for v in chunk]
    if op == _lib.REDUCE_SUM:
        t = sum(parts) & 0xFFFFFFFFFFFFFFFF
        return t - (1 << 64) if t >> 63 else t
    return max(parts, default=_INT64_MIN)


def sum_reduce(data, scheduler, batch_count: int = 1) -> int:
    """Sum of an integer view (int64 wrap-around, analytics.py:84-86); empty -> 0."""
    return _reduce(_check_view(data, batch_count), scheduler, batch_count, _lib.REDUCE_SUM)


def max_scan(data, scheduler, batch_count: int = 1) -> int:
    """Maximum of an integer view; empty view (and INT64_MIN) -> 0 (analytics.py:89-92)."""
    peak = _reduce(_check_view(data, batch_count), scheduler, batch_count, _lib.REDUCE_MAX)
    return 0 if peak == _INT64_MIN else peak


def _report_local(flat: FlatContainers) -> AggregateReport:
    """analyze_matrix on the calling thread's context (one rank of a group)."""
    w = _check_view(flat.weights, 1)
    fo = _lib.reduce_i64(_check_view(flat.out_degrees, 1), _lib.REDUCE_MAX)
    fi = _lib.reduce_i64(_check_view(flat.in_degrees, 1), _lib.REDUCE_MAX)
    return AggregateReport(
        valid_packets=_lib.reduce_i64(w, _lib.REDUCE_SUM),
        unique_links=len(flat.edges),
        unique_sources=len(flat.row_sums),
        max_fanout=0 if fo == _INT64_MIN else fo,
        unique_destinations=len(flat.col_sums),
        max_fanin=0 if fi == _INT64_MIN else fi,
    )


def analyze_matrix(flat: FlatContainers, scheduler, batch_count: int = 1) -> AggregateReport:
    """The six measures of one matrix from its flat containers (analytics.py:95-106)."""
    return AggregateReport(
        valid_packets=sum_reduce(flat.weights, scheduler, batch_count),
        unique_links=len(flat.edges),
        unique_sources=len(flat.row_sums),
        max_fanout=max_scan(flat.out_degrees, scheduler, batch_count),
        unique_destinations=len(flat.col_sums),
        max_fanin=max_scan(flat.in_degrees, scheduler, batch_count),
    )


def _totals6(reports) -> AggregateReport:
    return AggregateReport(
        valid_packets=sum(r.valid_packets for r in reports),
        unique_links=sum(r.unique_links for r in reports),
        unique_sources=sum(r.unique_sources for r in reports),
        max_fanout=max((r.max_fanout for r in reports), default=0),
        unique_destinations=sum(r.unique_destinations for r in reports),
        max_fanin=max((r.max_fanin for r in reports), default=0),
    )


def analyze_dataset(matrices, scheduler, batch_count: int = 1) -> tuple[list[AggregateReport], AggregateReport]:
    """Per-matrix reports plus dataset totals (analytics.py:109-130). With a device
    group the matrices are spread over its ranks by partition_even(len, G) (SURVEY.md
    8(e): windows shard with no collective), each rank building its containers and
    reports on its own device context concurrently."""
    if batch_count < 1:
        raise ValueError("batch_count must be >= 1")
    items = list(matrices)
    g = _group(scheduler)
    if g is None or g.resource_count == 1 or len(items) < 2:
        reports = []
        for item in items:
            flat = to_flat(item, device=_device_of(scheduler)) if isinstance(item, TrafficMatrix) else item
            reports.append(analyze_matrix(flat, scheduler, batch_count))
        return reports, _totals6(reports)

    def rank_part(r, lo, hi):
        return [_report_local(to_flat(it) if isinstance(it, TrafficMatrix) else it) for it in items[lo:hi]]

    reports = [rep for chunk in g.map_ranks(len(items), rank_part) for rep in chunk]
    return reports, _totals6(reports)


def oracle_analyze(window) -> AggregateReport:
    """The reference's independent cross-check (analytics.py:133-157): the six measures
    straight from raw pairs with host hash sets -- no matrix, no scheduler, and
    deliberately NOT the device hot path, so that comparing ``analyze_dataset`` /
    ``stats9`` against it compares two independent computations (as the reference's
    own tests do, tests/test_analytics.py:81-89). ``window``: a PacketStream (invalid
    packets skipped) or an iterable of (src, dst) pairs; any integer addresses."""
    if isinstance(window, PacketStream):
        keep = window.valid
        pairs = list(zip(window.src[keep].tolist(), window.dst[keep].tolist()))
    else:
        pairs = [(int(s), int(d)) for s, d in window]
    distinct = set(pairs)
    fanout: dict[int, int] = {}
    fanin: dict[int, int] = {}
    for s, d in distinct:  # every distinct link adds one to its row's and its column's nnz
        fanout[s] = fanout.get(s, 0) + 1
        fanin[d] = fanin.get(d, 0) + 1
    return AggregateReport(
        valid_packets=len(pairs),
        unique_links=len(distinct),
        unique_sources=len(fanout),
        max_fanout=max(fanout.values(), default=0),
        unique_destinations=len(fanin),
        max_fanin=max(fanin.values(), default=0),
    )


# ---------------------------------------------------------------------------
# the north-star hot path
# ---------------------------------------------------------------------------
def stats9(stream: PacketStream, device: int = 0, scheduler=None, batch_count: int = 1) -> Stats9:
    """Nine statistics of the matrix summed over all valid packets of ``stream``
    (= build_matrices(stream, len(stream)) -> to_flat -> analyze_matrix + 3 max_scan).

    ``scheduler``: a device group (make_group_scheduler(G)) shards the stream over its G
    ranks -- partition_even spans, ``batch_count`` H2D chunks per rank, owner(src) /
    owner(dst) exchanges inside libnmx.so (nmx_group_stats9_host); bit-identical for
    every G and batch_count."""
    if batch_count < 1:
        raise ValueError("batch_count must be >= 1")
    if len(stream) == 0:
        return Stats9.zero()
    g = _group(scheduler)
    if g is None:  # the stream's own int64 columns, narrowed inside the library (nmx_stats9_host_i64)
        if stream.address_space > 1 << 32:
            raise ValueError("address_space above 2^32 does not fit the 32-bit packet format")
        return Stats9(*_lib.stats9_i64(stream.src, stream.dst, stream.valid, stream.address_space, device=device))
    s, d, v = stream.wire()
    v = None if stream.valid.all() else v
    if g is not None and (g.resource_count > 1 or batch_count > 1):
        return Stats9(*g.native.stats9_host(s, d, v, stream.address_space, batch_count))
    if g is not None:
        with _lib.using(g.native.contexts[0]):
            return Stats9(*_lib.stats9(s, d, v, stream.address_space))
    return Stats9(*_lib.stats9(s, d, v, stream.address_space, device=device))


def analyze_summed(streams, device: int = 0, scheduler=None, batch_count: int = 1) -> Stats9:
    """Statistics of sum_t A_t over several streams (windows) of one address space:
    the element-wise sum of count matrices is the count matrix of the concatenated
    packets, so one device pass over all of them is exact."""
    streams = [streams] if isinstance(streams, PacketStream) else list(streams)
    if not streams:
        return Stats9.zero()
    space = max(s.address_space for s in streams)
    cat = PacketStream(np.concatenate([s.src for s in streams]), np.concatenate([s.dst for s in streams]),
                       np.concatenate([s.valid for s in streams]), space)
    return stats9(cat, device=device, scheduler=scheduler, batch_count=batch_count)


def _totals9(per) -> Stats9:
    sums = {0, 1, 3, 6}
    tot = [sum(r.astuple()[k] for r in per) if k in sums else max((r.astuple()[k] for r in per), default=0)
           for k in range(9)]
    return Stats9(*tot)


def analyze_windows(stream: PacketStream, window_size: int, device: int = 0,
                    scheduler=None) -> tuple[list[Stats9], Stats9]:
    """Per-window nine statistics with analyze_dataset totals (sums of the counting
    measures, maxima of the max measures; analytics.py:122-129). A device group
    spreads the windows over its ranks (partition_even(window_count, G)), no collective."""
    if window_size < 1:
        raise ValueError("window_size must be >= 1")
    if len(stream) == 0:
        return [], Stats9.zero()
    s, d, v = stream.wire()
    g = _group(scheduler)
    nwin = (len(stream) + window_size - 1) // window_size
    if g is None or g.resource_count == 1 or nwin < 2:
        if g is not None:
            with _lib.using(g.native.contexts[0]):
                rows = _lib.window_stats9(s, d, v, stream.address_space, window_size)
        else:
            rows = _lib.window_stats9(s, d, v, stream.address_space, window_size, device=device)
        per = [Stats9(*map(int, r)) for r in rows]
        return per, _totals9(per)

    def rank_part(r, lo, hi):
        if hi <= lo:
            return []
        a, b = lo * window_size, min(hi * window_size, len(stream))
        rows = _lib.window_stats9(s[a:b], d[a:b], v[a:b], stream.address_space, window_size)
        return [Stats9(*map(int, row)) for row in rows]

    per = [r for chunk in g.map_ranks(nwin, rank_part) for r in chunk]
    return per, _totals9(per)


def stats9_file(path, address_space: int | None = None, window_packets: int = 1 << 25, device: int = 0) -> Stats9:
    """Nine statistics of the matrix summed over every valid packet of a binary
    packet file (9-byte records, traffic.py:25, 370-388) -- read_packets ->
    build_matrices(stream, len(stream)) -> to_flat -> analyze_matrix + max_scan
    without materialising anything on the host: the file is read once into pinned
    memory and streamed to the GPU in windows of raw records, unpacked there
    (nmx_stream_records). ``address_space=None`` accepts any 32-bit address (the
    statistics do not depend on it); otherwise addresses >= address_space raise
    ValueError, like PacketStream."""
    import os

    size = os.path.getsize(path)
    if size % 9:
        raise ValueError(f"{path}: size {size} is not a whole number of 9-byte packet records")
    n = size // 9
    space = (1 << 32) if address_space is None else int(address_space)
    if n == 0:
        if space < 1:
            raise ValueError("address_space must be >= 1")
        return Stats9.zero()
    buf = _lib.PinnedArray(size, dtype=np.uint8)
    try:
        with open(path, "rb") as f:
            got = f.readinto(memoryview(buf.array))
        if got != size:
            raise OSError(f"{path}: short read ({got} of {size} bytes)")
        w = max(1, int(window_packets)) * 9
        windows = [buf.array[i:i + w] for i in range(0, size, w)]
        try:
            out = _lib.stream_records(windows, space, device)
        except _lib.NmxError as e:
            if "address_space" in str(e):
                raise ValueError(str(e)) from None
            raise
    finally:
        buf.close()
    return Stats9(*out)
