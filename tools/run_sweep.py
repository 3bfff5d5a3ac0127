"""C5: Llama-3.1-8B hyper-parameter sweep (64 configs) -- profile, calibrate, plan, place,
execute on the GPUs of one box, validate the executed trace, report the measured
wall-clock makespan beside the planner's prediction (reference cli.py:103-159).

  python tools/run_sweep.py [--gpus 8] [--plans balanced,reference,min] [--out gpurun_out/sweep.json]

With --gpus N and N visible GPUs the tool starts N ranks (torch.distributed.run, one
process per GPU; NCCL) and every rank executes the jobs placed on its device; the
makespan is the shared wall clock from the start barrier to the last job's end, and
the executed trace is re-checked with ``check_feasibility`` (reference
simulator.py:154-211).  With fewer GPUs than --gpus (a one-GPU box) one process
emulates the pool: each emulated device's jobs run back to back and the makespan is
the largest device busy time (``clock: device``, a lower bound).

1. profile: rank 0 trains 6 packs of 1 .. 16 configs for a few steps -> ProfileRecords;
2. calibrate: TimeModel per the reference least-squares fit with the B200 token term
   (grid-searched token_weight; load = r*b*s + w*b*s); degrees > 1 are costed d x the
   degree-1 job (tensor parallelism pays off only when a job does not fit one GPU);
3. plan: plan_jobs on the pool (memory model from the Llama-3.1-8B shapes) -- the B200
   balanced queue, the reference DTM queue, the Min-GPU baseline -- and their predicted
   makespans (``place`` reproduces the reference simulator's timeline);
4. execute: the engine runs every job for its full train_steps on its placed device.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import numpy as np  # noqa: E402

from paper_2508_02932_b200 import sweep as S  # noqa: E402
from paper_2508_02932_b200.model import PRESETS  # noqa: E402
from paper_2508_02932_b200.sweep.engine import execute, train_packed_job  # noqa: E402
from paper_2508_02932_b200.sweep.jobsplit import ACT_BYTES_PER_TOKEN  # noqa: E402


def grid(train_steps=50, seq=1024):
    tmpl = S.LoraConfig("t", rank=8, alpha=16.0, batch_size=1, learning_rate=1e-4, seq_len=seq, train_steps=train_steps)
    return S.enumerate_grid([5e-5, 1e-4, 2e-4, 4e-4], [1, 2], [8, 16, 32, 64], [16.0, 64.0], tmpl)


def calibrate(configs, by_id, model, pool, steps):
    rng = np.random.default_rng(0)
    packs = [[0], [5, 17], list(range(0, 64, 16)), list(range(3, 64, 8)), list(rng.choice(64, 12, replace=False)),
             list(range(1, 64, 4))]
    profiles = []
    for p in packs:
        job = S.make_job([configs[i].id for i in p], 1, S.TimeModel(coeffs={1: (1.0, 0.0)}),
                         S.MemoryContext(model, pool, configs))
        import torch
        dev = f"cuda:{torch.cuda.current_device()}"   # the engine's device key: the base weights are shared
        _, _, it, _ = train_packed_job(job, by_id, "llama-3.1-8b", dev, steps_override=steps)
        cf = [by_id[c] for c in job.configs]
        profiles.append(S.ProfileRecord(1, tuple(c.rank for c in cf), tuple(c.batch_size for c in cf), 1024, it))
        print(f"profile: {len(p)} configs, {sum(c.batch_size for c in cf)} seqs -> {it:.3f} s/iter", flush=True)
    best = None
    for w in (0.0, 4.0, 16.0, 64.0, 256.0, 1024.0):
        try:
            tm1 = S.calibrate_time_model(profiles, token_weight=w, max_rel_rmse=1.0)
        except S.CalibrationError:
            continue
        if best is None or tm1.fit_rel_rmse[1] < best.fit_rel_rmse[1]:
            best = tm1
    b1, m1 = best.params(1)
    return {"base_s": b1, "marginal_s": m1, "token_weight": best.token_weight, "rel_rmse": best.fit_rel_rmse[1],
            "profiles": [dict(ranks=list(p.packed_ranks), batch_sizes=list(p.packed_batch_sizes),
                              iter_time_s=p.iter_time_s) for p in profiles]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--steps", type=int, default=None, help="override every job's train_steps (default: full)")
    ap.add_argument("--plans", default="balanced,reference,min")
    ap.add_argument("--mem-gb", type=float, default=178.0)
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    ndev = torch.cuda.device_count()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and ndev >= args.gpus:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        raise SystemExit(subprocess.call([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                          f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                          f"--master-port={port}", __file__, *sys.argv[1:]]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, ndev))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local % max(1, ndev)))

    def gather(obj):
        if world == 1:
            return [obj]
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    t_start = time.perf_counter()
    cfg = PRESETS["llama-3.1-8b"]
    configs = grid()
    if args.steps:
        configs = [S.LoraConfig(c.id, rank=c.rank, alpha=c.alpha, batch_size=c.batch_size,
                                learning_rate=c.learning_rate, seq_len=c.seq_len, train_steps=args.steps)
                   for c in configs]
    by_id = {c.id: c for c in configs}
    half = ACT_BYTES_PER_TOKEN / 2 / 2
    model = S.model_spec_from_config(cfg, c_prec=2, act_coeffs=(0.0, half, half), state_bytes=S.STATE_BYTES_PLORA)
    pool = S.GpuPool(args.gpus, int(args.mem_gb * 1e9), load_factor=0.9)

    cal = calibrate(configs, by_id, model, pool, args.profile_steps) if rank == 0 else None
    cal = gather(cal)[0]
    b1, m1 = cal["base_s"], cal["marginal_s"]
    tm = S.TimeModel(coeffs={d: (b1 * d, m1 * d) for d in (1, 2, 4, 8) if d <= args.gpus},
                     token_weight=cal["token_weight"])
    if rank == 0:
        print(f"calibrated: base {b1:.4f} s, marginal {m1:.3e} s/load, token_weight {cal['token_weight']}, "
              f"rel rmse {cal['rel_rmse']:.3f}", flush=True)
    mem = S.MemoryContext(model, pool, configs)
    queues = {"balanced": S.plan_jobs(args.gpus, configs, tm, mem, balance=True),
              "reference": S.plan_jobs(args.gpus, configs, tm, mem),
              "min": S.min_gpu_queue(configs, args.gpus, tm, mem)}
    out = {"configs": len(configs), "gpus": args.gpus, "processes": world, "time_model": cal, "plans": {}}
    for name in args.plans.split(","):
        q = queues[name]
        pred = S.place(q, args.gpus).makespan
        rep = execute(q, configs, args.gpus, rank=rank, world=world, all_gather=gather, pool=pool)
        bound = S.ar_bound(rep["trace"])
        out["plans"][name] = {
            "jobs": len(q.jobs()), "degrees": sorted({j.degree for j in q.jobs()}),
            "predicted_makespan_s": pred, "measured_makespan_s": rep["makespan_s"], "clock": rep["clock"],
            "violations": rep["violations"], "ar_bound": bound.bound,
            "busy_s": rep["busy_s"],
            "trace": [dict(job=j.job_id, configs=len(j.configs), degree=j.degree, devices=list(j.devices),
                           start_s=round(j.start_s, 3), duration_s=round(j.duration_s, 3),
                           predicted_s=round(j.predicted_s, 3)) for j in rep["trace"].jobs]}
        if rank == 0:
            print(f"{name}: {len(q.jobs())} jobs, predicted {pred:.1f} s, measured {rep['makespan_s']:.1f} s "
                  f"({rep['clock']} clock), violations {len(rep['violations'])}", flush=True)
    if rank == 0:
        out["wall_s"] = time.perf_counter() - t_start
        if "balanced" in out["plans"] and "min" in out["plans"]:
            out["speedup_vs_min_gpu_measured"] = (out["plans"]["min"]["measured_makespan_s"]
                                                  / out["plans"]["balanced"]["measured_makespan_s"])
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps({k: {kk: v[kk] for kk in ("jobs", "predicted_makespan_s", "measured_makespan_s", "clock",
                                                     "violations")} for k, v in out["plans"].items()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
