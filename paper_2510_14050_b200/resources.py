"""Execution resources: a group of B200 ranks replaces the reference's thread-pool
"devices" (resources.py:95-159 of /root/reference/pkg/src/netmeter).

``make_group_scheduler(G)`` returns a ``DeviceGroup`` whose ``resource_count`` is
G. Rank r runs on CUDA device ``r mod (visible devices)`` with its OWN library
context (stream + workspace, ``nmx_group`` in include/nmx.h), so G ranks on G
B200s run concurrently and G ranks on fewer devices are virtual ranks sharing a
device. The analytics entry points dispatch through the group:

* ``stats9`` / ``analyze_summed``: the sharded owner(src) / owner(dst) pipeline
  runs inside libnmx.so (``nmx_group_stats9_host``), one host thread per rank,
  exchanges as peer copies;
* ``analyze_dataset`` / ``analyze_windows``: windows -> ranks by
  ``partition_even(window_count, G)`` (partitioning.py:62-70), no collective;
* ``sum_reduce`` / ``max_scan``: the view -> ranks by ``partition_even``, each
  rank's span in ``batch_count`` chunks (batch_table, partitioning.py:89-98),
  partials combined on the host like the reference's per-resource slots
  (analytics.py:54-81).

The device group is created on first use, so building schedulers (and their
argument errors) works without a GPU. ``run_bulk`` keeps the SchedulerLike
contract (senders.py:32-38) for host tasks: every index exactly once, spans of
``partition_even`` run concurrently, one thread per rank.
"""

from __future__ import annotations

import threading

from .partitioning import partition_even


class DeviceGroup:
    """``resource_count`` ranks; rank r maps to CUDA device ``devices[r]``."""

    def __init__(self, count: int, workers_per_resource: int = 1):
        if count < 1:
            raise ValueError("group needs at least one device")
        self._count = int(count)
        self.workers_per_resource = int(workers_per_resource)
        self._group = None
        self._lock = threading.Lock()

    @property
    def resource_count(self) -> int:
        return self._count

    @property
    def devices(self) -> list[int]:
        from . import _lib

        nd = max(1, _lib.device_count())
        return [r % nd for r in range(self._count)]

    @property
    def device(self) -> int:
        return 0

    @property
    def native(self):
        """The libnmx device group (``_lib.Group``), created on first use."""
        with self._lock:
            if self._group is None:
                from . import _lib

                self._group = _lib.Group(self.devices)
            return self._group

    def map_ranks(self, n_items: int, fn) -> list:
        """Call ``fn(rank, lo, hi)`` for each rank's ``partition_even`` span of
        ``n_items`` items, concurrently (one host thread per rank, bound to the rank's
        context); returns the per-rank results in rank order. The first failure is
        re-raised after every rank has finished."""
        from . import _lib

        spans = partition_even(n_items, self._count).spans
        if self._count == 1:
            with _lib.using(self.native.contexts[0]):
                return [fn(0, 0, n_items)]
        out: list = [None] * self._count
        errs: list = []

        def work(r, lo, hi):
            try:
                with _lib.using(self.native.contexts[r]):
                    out[r] = fn(r, lo, hi)
            except BaseException as e:  # noqa: BLE001 - re-raised below
                errs.append(e)

        self.native  # create before the threads race for it
        th = [threading.Thread(target=work, args=(r, off, off + ln)) for r, (off, ln) in enumerate(spans)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        return out

    def run_bulk(self, size: int, task, payload: tuple) -> None:
        """SchedulerLike.run_bulk (senders.py:32-38): task(i, resource_id, *payload) exactly
        once per index, indices split evenly and contiguously over the resources
        (resources.py:107-113), the resources' spans running concurrently."""
        if size < 0:
            raise ValueError("bulk size must be >= 0")
        spans = partition_even(size, self._count).spans
        errs: list = []

        def work(rid, off, ln):
            try:
                for i in range(off, off + ln):
                    task(i, rid, *payload)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)

        th = [threading.Thread(target=work, args=(rid, off, ln)) for rid, (off, ln) in enumerate(spans) if ln]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]

    def close(self) -> None:
        with self._lock:
            if self._group is not None:
                self._group.close()
                self._group = None

    def __enter__(self) -> "DeviceGroup":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def make_inline_scheduler() -> DeviceGroup:
    return DeviceGroup(1)


def make_pool_scheduler(workers: int) -> DeviceGroup:
    """One device; ``workers`` is the host-thread count the reference's pool would use
    (kept for run_bulk semantics; device work runs on the rank's stream)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return DeviceGroup(1, workers)


def make_group_scheduler(resources, workers_per_resource: int | None = None) -> DeviceGroup:
    """resources.py:139-159 signature: a rank count, or a list (one entry per rank,
    each the worker count of the reference's per-resource pool)."""
    if isinstance(resources, int):
        if resources < 1:
            raise ValueError("resource count must be >= 1")
        return DeviceGroup(resources, workers_per_resource or 1)
    if workers_per_resource is not None:
        raise ValueError("pass workers_per_resource only with a resource count")
    specs = list(resources)
    if not specs:
        raise ValueError("group needs at least one pool spec")
    for w in specs:
        if int(w) < 1:
            raise ValueError("workers must be >= 1")
    return DeviceGroup(len(specs), max(int(w) for w in specs))
