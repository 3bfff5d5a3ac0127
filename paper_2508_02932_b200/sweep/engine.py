"""Execution engine: run a planned JobQueue on the GPUs of one box.

PLoRA's "LoRA Execution Engine" (absent from the reference,
SPEC.md:550) closes the planner loop:

  plan_jobs -> place (devices) -> one process per GPU runs the jobs placed on it,
  each job = a packed multi-LoRA training run (PackedLoraTrainer) for the longest
  member's train_steps -> measured per-job times and ProfileRecords -> a B200
  calibrated TimeModel (calibrate_time_model) -> re-plan / report makespan.

Multi-GPU: jobs are independent, so ranks never exchange data between jobs; the
collectives are the final gather of job records / per-device busy time over
torch.distributed (NCCL on the box, gloo in the CPU tests) and, inside a job of
degree d > 1, the tensor-parallel all-reduces of that job's d ranks (tp.py,
config C4): ``execute`` creates one process group per distinct device set of the
queue (every rank, same order), and each member rank trains its Megatron shard
of the job.  TP jobs need one process per GPU (world == gpu_count).

``run_job`` is injectable so the host-side scheduling logic is testable without
a GPU (tests/test_engine.py runs it under gloo, world size 2).
"""

from __future__ import annotations

import hashlib
import json
import time
from dataclasses import asdict, dataclass
from typing import Callable, Sequence

from .planner import JobQueue, Placement, place
from .trace import ScheduleTrace, TraceJob, check_feasibility
from .workload import GpuPool, LoraConfig, ProfileRecord


@dataclass(frozen=True)
class JobRecord:
    """One job as one device ran it.  ``start_s``/``end_s``: seconds since the shared
    start barrier of all ranks (wall clock); ``device_start_s``: the device's own busy
    clock at the job's start (when one process emulates several devices back to back,
    this is the job's start on the emulated device); ``train_s``: the timed steps only."""
    job_id: str
    device: int
    configs: tuple
    steps: int
    start_s: float
    end_s: float
    device_start_s: float
    train_s: float
    iter_time_s: float
    losses: tuple = ()

    @property
    def duration_s(self) -> float:
        return self.end_s - self.start_s


def rank_schedule(queue: JobQueue, placement: Placement, rank: int) -> list:
    """Jobs this rank (device) executes, in planned start order."""
    mine = [j for j in queue.jobs() if rank in placement.devices[j.id]]
    return sorted(mine, key=lambda j: (placement.start_s[j.id], j.id))


_BASE_CACHE: dict = {}


def _base(model_name: str, device: str):
    """Frozen base weights are shared by every job a process runs on a device."""
    from ..model import PRESETS, BaseWeights

    key = (model_name, device)
    if key not in _BASE_CACHE:
        _BASE_CACHE[key] = BaseWeights(PRESETS[model_name], device)
    return _BASE_CACHE[key]


def train_packed_job(job, configs_by_id: dict, model_name: str, device: str, steps_override: int | None = None,
                     warmup: int = 1, tp=None, checkpoint_dir=None) -> tuple:
    """Run one packed job on ``device`` (its TP shard when ``tp`` is a communicator over
    the job's ranks): returns (steps, seconds, mean iteration seconds, losses).  With
    ``checkpoint_dir`` every configuration's adapter is written to the checkpoint pool
    (checkpoint.py) when the job ends."""
    import torch

    from ..model import PRESETS, AdapterSpec, PackedLoraTrainer

    cfgs = [configs_by_id[c] for c in job.configs]
    seq = max(c.seq_len for c in cfgs)
    specs = [AdapterSpec(rank=c.rank, alpha=c.alpha, batch=c.batch_size, lr=c.learning_rate) for c in cfgs]
    seeds = [int(hashlib.sha256(c.id.encode()).hexdigest()[:8], 16) for c in cfgs]
    base = _base(model_name, device) if tp is None or tp.world == 1 else None   # TP shards: per-job base slices
    trainer = PackedLoraTrainer(PRESETS[model_name], specs, seq, device=device, base=base, adapter_seeds=seeds, tp=tp)
    steps = steps_override or max(c.train_steps for c in cfgs)
    tokens = trainer.synthetic_tokens().to(device)
    for _ in range(warmup):
        trainer.step(tokens)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        losses = trainer.step(tokens)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out = tuple(float(x) for x in losses.tolist())
    if checkpoint_dir is not None:
        from ..checkpoint import save_adapter

        for i, c in enumerate(cfgs):
            save_adapter(trainer, i, checkpoint_dir, config_id=c.id, extra={"job_id": job.id, "degree": job.degree})
    del trainer
    torch.cuda.empty_cache()
    return steps, dt, dt / steps, out


def tp_groups(queue: JobQueue, placement: Placement, world: int, gpu_count: int,
              new_group: Callable | None = None) -> dict:
    """One communicator per distinct device set of the queue's degree > 1 jobs, created on
    every rank in the same (sorted) order -- torch.distributed.new_group is collective."""
    sets = sorted({placement.devices[j.id] for j in queue.jobs() if j.degree > 1})
    if not sets:
        return {}
    if world != gpu_count:
        raise NotImplementedError("tensor-parallel jobs need one process per GPU (world == gpu_count)")
    if new_group is None:
        import torch.distributed as dist

        from ..tp import DistComm

        def new_group(ranks):
            g = dist.new_group(list(ranks))
            return DistComm(g) if dist.get_rank() in ranks else None
    out = {}
    for devs in sets:
        comm = new_group(devs)
        if comm is not None:
            out[devs] = comm
    return out


def _device_guard(dev: int):
    """Run a job with its device current: libplora launches on the current device's
    stream, so tensors of cuda:dev must be used with dev current."""
    import contextlib

    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.device(dev % max(1, torch.cuda.device_count()))
    except Exception:  # pragma: no cover
        pass
    return contextlib.nullcontext()


def execute(queue: JobQueue, configs: Sequence[LoraConfig], gpu_count: int, *, rank: int = 0, world: int = 1,
            model_name: str = "llama-3.1-8b", run_job: Callable | None = None,
            steps_override: int | None = None, all_gather: Callable | None = None,
            new_group: Callable | None = None, checkpoint_dir=None, pool: GpuPool | None = None) -> dict:
    """Execute this rank's share of the queue and return the report of the whole queue.

    One process per GPU (world == gpu_count): rank r runs the jobs placed on device r in
    planned start order, with device r current; all ranks start from one barrier
    (``all_gather``) and every job records its wall-clock start / end since that
    barrier, so ``makespan_s`` is the measured wall-clock makespan of the queue.  A
    degree-d job starts on all d ranks together (its process group synchronises them).
    With fewer processes than GPUs (one box with one GPU emulating a larger pool), a rank
    drives every device = rank (mod world) back to back; the trace then uses each
    device's busy clock (``clock == "device"``, a lower bound of the real makespan).
    The executed trace is checked against the queue with ``check_feasibility``
    (reference simulator.py:154-211); violations are reported, not raised."""
    placement = place(queue, gpu_count)
    groups = tp_groups(queue, placement, world, gpu_count, new_group)
    by_id = {c.id: c for c in configs}
    devices = list(range(rank, gpu_count, world))
    emulated = world < gpu_count
    if all_gather is not None:
        all_gather(None)                      # shared start barrier
    t0 = time.perf_counter()
    records = []
    for dev in devices:
        clock = 0.0
        for job in rank_schedule(queue, placement, dev):
            comm = groups.get(placement.devices[job.id])
            extra = {"tp": comm} if comm is not None else {}
            s = time.perf_counter() - t0
            with _device_guard(dev):
                if run_job is None:
                    steps, dt, it, losses = train_packed_job(job, by_id, model_name, _cuda(dev), steps_override,
                                                             checkpoint_dir=checkpoint_dir, **extra)
                else:
                    steps, dt, it, losses = run_job(job, by_id, dev, **extra)
            e = time.perf_counter() - t0
            records.append(JobRecord(job.id, dev, job.configs, steps, s, e, clock, dt, it, tuple(losses)))
            clock += e - s
    local = {"records": [asdict(r) for r in records]}
    gathered = all_gather(local) if all_gather is not None else [local]
    all_records = [JobRecord(**{**r, "configs": tuple(r["configs"]), "losses": tuple(r["losses"])})
                   for g in gathered for r in g["records"]]
    busy: dict = {}
    for r in all_records:
        busy[r.device] = busy.get(r.device, 0.0) + r.duration_s
    trace = executed_trace(queue, all_records, gpu_count, clock="device" if emulated else "wall")
    violations = check_feasibility(trace, queue, pool)
    # one profile record per job (a TP job reports from each of its ranks: keep the slowest)
    degree = {j.id: j.degree for j in queue.jobs()}
    per_job: dict = {}
    for r in all_records:
        if r.job_id not in per_job or r.iter_time_s > per_job[r.job_id].iter_time_s:
            per_job[r.job_id] = r
    profiles = [ProfileRecord(degree[r.job_id], tuple(by_id[c].rank for c in r.configs),
                              tuple(by_id[c].batch_size for c in r.configs),
                              max(by_id[c].seq_len for c in r.configs), r.iter_time_s)
                for _, r in sorted(per_job.items())]
    return {"records": all_records, "profiles": profiles, "makespan_s": trace.makespan, "clock": trace.clock,
            "busy_s": busy, "placement": placement, "trace": trace, "violations": violations}


def executed_trace(queue: JobQueue, records: Sequence[JobRecord], gpu_count: int, clock: str = "wall"
                   ) -> ScheduleTrace:
    """The schedule that ran: one TraceJob per executed job id, on every device that ran
    it, from the earliest start to the latest end over those devices (wall clock), or on
    the device busy clocks (``clock == "device"``)."""
    predicted = {j.id: j for j in queue.jobs()}
    by_job: dict = {}
    for r in records:
        by_job.setdefault(r.job_id, []).append(r)
    jobs = []
    for jid, rs in sorted(by_job.items(), key=lambda kv: (min(r.start_s for r in kv[1]), kv[0])):
        if clock == "wall":
            s, e = min(r.start_s for r in rs), max(r.end_s for r in rs)
        else:
            s = min(r.device_start_s for r in rs)
            e = max(r.device_start_s + r.duration_s for r in rs)
        p = predicted.get(jid)
        jobs.append(TraceJob(job_id=jid, configs=tuple(rs[0].configs), degree=p.degree if p else len(rs),
                             start_s=s, duration_s=e - s, devices=tuple(sorted({r.device for r in rs})),
                             predicted_s=p.predicted_time if p else 0.0))
    return ScheduleTrace(jobs=tuple(jobs), makespan=max((j.end_s for j in jobs), default=0.0),
                         gpu_count=gpu_count, clock=clock)


def _cuda(dev: int) -> str:
    return f"cuda:{dev % max(1, _ndev())}"


def _ndev() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # pragma: no cover
        return 1


def report_json(rep: dict) -> str:
    return json.dumps({"makespan_s": rep["makespan_s"], "clock": rep["clock"], "busy_s": rep["busy_s"],
                       "violations": rep["violations"], "jobs": [asdict(r) for r in rep["records"]]}, indent=1)
