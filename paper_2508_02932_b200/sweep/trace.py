"""Executed schedules and their validity check.

The engine (engine.py) records, for every job of a queue, when and on which devices it
actually ran; ``check_feasibility`` re-derives the scheduling constraints from that
record, as the reference does for its simulated traces (pkg/src/lorasweep/
simulator.py:154-211): every configuration planned and run exactly once, each job on
``degree`` distinct in-pool devices, never two jobs on one device at the same time,
no job over the per-device memory budget, the makespan equal to the last completion.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import combinations

from .planner import JobQueue
from .workload import GpuPool


@dataclass(frozen=True)
class TraceJob:
    """One executed job (reference simulator.py:44-64 field names)."""

    job_id: str
    configs: tuple
    degree: int
    start_s: float
    duration_s: float
    devices: tuple
    predicted_s: float

    @property
    def end_s(self) -> float:
        return self.start_s + self.duration_s

    @property
    def drift_s(self) -> float:
        return self.duration_s - self.predicted_s


@dataclass(frozen=True)
class ScheduleTrace:
    jobs: tuple
    makespan: float
    gpu_count: int
    clock: str = "wall"      # "wall": shared wall clock of one process per GPU; "device": per-device busy clock


def check_feasibility(trace: ScheduleTrace, queue: JobQueue, pool: GpuPool | None = None) -> list:
    """Constraint violations of ``trace`` as an execution of ``queue`` (empty = valid).
    ``pool`` defaults to the trace's GPU count with no memory budget."""
    gpu_count = pool.gpu_count if pool is not None else trace.gpu_count
    budget = pool.memory_budget if pool is not None else math.inf
    planned = {j.id: j for j in queue.jobs()}
    out = []

    def count(jobs):
        c: dict = {}
        for j in jobs:
            for cid in j.configs:
                c[cid] = c.get(cid, 0) + 1
        return c

    want, got = count(queue.jobs()), count(trace.jobs)
    for cid in sorted(want):
        if want[cid] != 1:
            out.append(f"configuration '{cid}' planned {want[cid]} times")
        if got.get(cid, 0) != 1:
            out.append(f"configuration '{cid}' executed {got.get(cid, 0)} times (expected once)")
    out += [f"configuration '{cid}' executed but never planned" for cid in sorted(set(got) - set(want))]

    for j in trace.jobs:
        if len(set(j.devices)) != len(j.devices):
            out.append(f"job '{j.job_id}' repeats a device")
        if len(j.devices) != j.degree:
            out.append(f"job '{j.job_id}' ran on {len(j.devices)} devices but its degree is {j.degree}")
        out += [f"job '{j.job_id}' device {d} outside the pool of {gpu_count}"
                for d in j.devices if not 0 <= d < gpu_count]
        if j.start_s < 0:
            out.append(f"job '{j.job_id}' starts before time zero")
        p = planned.get(j.job_id)
        if p is None:
            out.append(f"job '{j.job_id}' is not in the queue")
        elif p.predicted_memory > budget:
            out.append(f"job '{j.job_id}' needs {p.predicted_memory} bytes per device, budget is {budget:.0f}")

    for a, b in combinations(trace.jobs, 2):
        shared = sorted(set(a.devices) & set(b.devices))
        if shared and a.start_s < b.end_s and b.start_s < a.end_s:
            out.append(f"jobs '{a.job_id}' and '{b.job_id}' overlap on device(s) {shared}")

    last = max((j.end_s for j in trace.jobs), default=0.0)
    if not math.isclose(trace.makespan, last, rel_tol=1e-12, abs_tol=1e-9):
        out.append(f"makespan {trace.makespan} differs from the last completion {last}")
    return out
