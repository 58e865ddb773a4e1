"""Measured step reports with the reference's schema (pkg/src/ralp/simulator.py:163-282).

`StepBreakdown` keeps the four categories of the paper's timeline accounting
(worker computation, PS computation, memcopy, communication); `JobReport`
derives avg_step_time (mean over steps of the slowest worker), images_per_sec
(W*b / avg_step_time) and comm_fraction exactly as the reference does.  The
measured backend adds `losses` (one per step, PS rank).

VENDORED API MIRROR (attribution): this module follows the reference `ralp` package's own code for
the same surface closely -- same classes, checks, error messages and arithmetic -- because north_star
makes that planner API the drop-in surface and its outputs must match the reference bit-exactly
(tests/test_planner_golden.py pins them to the unmodified reference).  It is not original work and
it is not on the GPU path; the executor accepts the reference's own objects as well
(executor.py `_kv`).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field


@dataclass(frozen=True)
class StepBreakdown:
    job: str
    step: int
    worker_computation: tuple[float, ...]
    ps_computation: tuple[float, ...]
    memcopy: tuple[float, ...]
    communication: tuple[float, ...]

    def step_duration(self, worker: int) -> float:
        return (self.worker_computation[worker] + self.ps_computation[worker] + self.memcopy[worker]
                + self.communication[worker])

    @property
    def step_durations(self) -> tuple[float, ...]:
        return tuple(self.step_duration(w) for w in range(len(self.worker_computation)))

    @property
    def avg_step_time(self) -> float:
        d = self.step_durations
        return sum(d) / len(d)

    @property
    def max_step_time(self) -> float:
        return max(self.step_durations)

    def to_dict(self) -> dict:
        return {"job": self.job, "step": self.step, "worker_computation": list(self.worker_computation),
                "ps_computation": list(self.ps_computation), "memcopy": list(self.memcopy),
                "communication": list(self.communication), "avg_step_time": self.avg_step_time,
                "max_step_time": self.max_step_time}


@dataclass(frozen=True)
class JobReport:
    job: str
    strategy: str
    worker_count: int
    batch_size: int
    steps: tuple[StepBreakdown, ...]
    bytes_on_wire_per_step: int
    losses: tuple[float, ...] = field(default=())

    @property
    def avg_step_time(self) -> float:
        return sum(s.max_step_time for s in self.steps) / len(self.steps)

    @property
    def images_per_sec(self) -> float:
        return self.worker_count * self.batch_size / self.avg_step_time

    @property
    def comm_fraction(self) -> float:
        comm = sum(sum(s.communication) for s in self.steps)
        total = sum(sum(s.step_durations) for s in self.steps)
        return comm / total if total > 0 else 0.0

    def to_dict(self) -> dict:
        return {"job": self.job, "strategy": self.strategy, "worker_count": self.worker_count,
                "batch_size": self.batch_size, "avg_step_time": self.avg_step_time,
                "images_per_sec": self.images_per_sec, "comm_fraction": self.comm_fraction,
                "bytes_on_wire_per_step": self.bytes_on_wire_per_step, "losses": list(self.losses),
                "steps": [s.to_dict() for s in self.steps]}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)
