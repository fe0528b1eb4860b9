"""Benchmark result records (mirror of bench.py:14-56 of the reference).

Two clocks per run: analysis time covers only the statistics pipeline,
end-to-end time covers the whole run including matrix loading and container
construction. Packet rate is packets per second of end-to-end time and always
recomputes exactly from the stored fields.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass(frozen=True)
class RunConfig:
    """Knobs of one benchmark run; None for values unknown at analyze time."""

    resources: int
    workers_per_resource: int | None = None
    batch_count: int = 1
    window_size: int | None = None
    packet_count: int | None = None
    seed: int | None = None

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass(frozen=True)
class BenchResult:
    analysis_time: float
    end_to_end_time: float
    packet_count: int
    packet_rate: float
    config: RunConfig

    def __post_init__(self):
        if self.analysis_time > self.end_to_end_time:
            raise ValueError("analysis_time cannot exceed end_to_end_time")

    @classmethod
    def from_times(cls, analysis_time: float, end_to_end_time: float, packet_count: int,
                   config: RunConfig) -> "BenchResult":
        return cls(analysis_time=analysis_time, end_to_end_time=end_to_end_time, packet_count=packet_count,
                   packet_rate=packet_count / end_to_end_time, config=config)

    def to_dict(self) -> dict:
        out = asdict(self)
        out["config"] = self.config.to_dict()
        return out
