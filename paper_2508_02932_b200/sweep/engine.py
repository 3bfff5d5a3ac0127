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
from .workload import LoraConfig, ProfileRecord


@dataclass(frozen=True)
class JobRecord:
    job_id: str
    device: int
    configs: tuple
    steps: int
    start_s: float
    duration_s: float
    iter_time_s: float
    losses: tuple = ()


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


def execute(queue: JobQueue, configs: Sequence[LoraConfig], gpu_count: int, *, rank: int = 0, world: int = 1,
            model_name: str = "llama-3.1-8b", run_job: Callable | None = None,
            steps_override: int | None = None, all_gather: Callable | None = None,
            new_group: Callable | None = None, checkpoint_dir=None) -> dict:
    """Execute this rank's share of the queue.  Returns a report with the per-job records
    (gathered from every rank when ``all_gather`` is given), profile records, the
    measured makespan (max over ranks of the per-device busy time) and the placement."""
    placement = place(queue, gpu_count)
    groups = tp_groups(queue, placement, world, gpu_count, new_group)
    by_id = {c.id: c for c in configs}
    devices = list(range(rank, gpu_count, world))   # a rank drives every device = rank (mod world)
    records = []
    t_dev = {}
    for dev in devices:
        clock = 0.0
        for job in rank_schedule(queue, placement, dev):
            comm = groups.get(placement.devices[job.id])
            extra = {"tp": comm} if comm is not None else {}
            if run_job is None:
                steps, dt, it, losses = train_packed_job(job, by_id, model_name, f"cuda:{dev % max(1, _ndev())}",
                                                         steps_override, checkpoint_dir=checkpoint_dir, **extra)
            else:
                steps, dt, it, losses = run_job(job, by_id, dev, **extra)
            records.append(JobRecord(job.id, dev, job.configs, steps, clock, dt, it, tuple(losses)))
            clock += dt
        t_dev[dev] = clock
    local = {"records": [asdict(r) for r in records], "busy_s": t_dev}
    gathered = all_gather(local) if all_gather is not None else [local]
    all_records = [JobRecord(**{**r, "configs": tuple(r["configs"]), "losses": tuple(r["losses"])})
                   for g in gathered for r in g["records"]]
    busy = {int(k): v for g in gathered for k, v in g["busy_s"].items()}
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
    return {"records": all_records, "profiles": profiles, "makespan_s": max(busy.values(), default=0.0),
            "busy_s": busy, "placement": placement}


def _ndev() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # pragma: no cover
        return 1


def report_json(rep: dict) -> str:
    return json.dumps({"makespan_s": rep["makespan_s"], "busy_s": rep["busy_s"],
                       "jobs": [asdict(r) for r in rep["records"]]}, indent=1)
