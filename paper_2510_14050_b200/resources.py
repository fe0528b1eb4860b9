"""Execution resources: a group of B200s replaces the reference's thread-pool
"devices" (resources.py:95-159). Only the scheduler *interface* is mirrored
(``resource_count``, ``run_bulk``, context manager, the ``make_*`` factories and
their argument errors); device work never goes through ``run_bulk`` -- the
analytics entry points launch libnmx.so kernels on ``device`` directly.
"""

from __future__ import annotations

from .partitioning import partition_even


class DeviceGroup:
    """``resource_count`` GPUs; resource r maps to CUDA device ``devices[r]``."""

    def __init__(self, devices: list[int]):
        if not devices:
            raise ValueError("group needs at least one device")
        self.devices = list(devices)

    @property
    def resource_count(self) -> int:
        return len(self.devices)

    @property
    def device(self) -> int:
        return self.devices[0]

    def run_bulk(self, size: int, task, payload: tuple) -> None:
        """SchedulerLike.run_bulk (senders.py:32-38): task(i, resource_id, *payload) exactly
        once per index, indices split evenly and contiguously over the resources
        (resources.py:107-113). Host-side compatibility for user tasks."""
        if size < 0:
            raise ValueError("bulk size must be >= 0")
        for rid, (off, ln) in enumerate(partition_even(size, self.resource_count).spans):
            for i in range(off, off + ln):
                task(i, rid, *payload)

    def close(self) -> None:
        pass

    def __enter__(self) -> "DeviceGroup":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


def make_inline_scheduler() -> DeviceGroup:
    return DeviceGroup([0])


def make_pool_scheduler(workers: int) -> DeviceGroup:
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return DeviceGroup([0])


def make_group_scheduler(resources, workers_per_resource: int | None = None) -> DeviceGroup:
    """resources.py:139-159 signature: a count, or a list (one entry per resource)."""
    if isinstance(resources, int):
        if resources < 1:
            raise ValueError("resource count must be >= 1")
        count = resources
    else:
        if workers_per_resource is not None:
            raise ValueError("pass workers_per_resource only with a resource count")
        specs = list(resources)
        if not specs:
            raise ValueError("group needs at least one pool spec")
        count = len(specs)
    return DeviceGroup(list(range(count)))
