"""Execution-engine host logic (planner placement -> per-rank job lists -> gathered
records / makespan) under torch.distributed gloo, world size 2, on CPU.  The GPU
job runner is replaced by a deterministic fake; tests/test_gpu_engine.py runs real jobs."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_02932_b200 import sweep as S
from paper_2508_02932_b200.sweep.engine import execute, rank_schedule


def _instance(n=10, G=4):
    model = S.ModelSpec("m", 1, (S.TargetModule("q", 1 << 20, 1 << 20),), 0, 2)
    configs = [S.LoraConfig(f"c{i:02d}", rank=8 * (1 + i % 3), alpha=16.0, batch_size=1 + i % 2,
                            learning_rate=1e-4, seq_len=16, train_steps=2 + i % 3) for i in range(n)]
    per = S.lora_state_memory(configs[0], model, S.ShardingSpec()).total_bytes
    pool = S.GpuPool(G, int(per * 4.5))
    tm = S.TimeModel(coeffs={1: (1.0, 1e-4), 2: (1.0, 1e-4), 4: (1.0, 1e-4)})   # no TP speedup -> degree 1
    mem = S.MemoryContext(model, pool, configs)
    return configs, S.plan_jobs(G, configs, tm, mem), tm


def fake_run(job, by_id, dev):
    import time
    steps = max(by_id[c].train_steps for c in job.configs)
    it = 0.1 + 0.01 * len(job.configs)
    time.sleep(0.002 * len(job.configs))      # wall time the engine records
    return steps, steps * it, it, [1.0] * len(job.configs)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(obj):
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    configs, queue, _ = _instance()
    rep = execute(queue, configs, 4, rank=rank, world=world, run_job=fake_run, all_gather=gather)
    out[rank] = (rep["makespan_s"], sorted((r.job_id, r.device) for r in rep["records"]), rep["busy_s"],
                 rep["violations"], rep["clock"])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_engine_two_ranks_gloo():
    configs, queue, _ = _instance()
    assert all(j.degree == 1 for j in queue.jobs())
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r0, r1 = out[0], out[1]
    assert r0 == r1                                       # every rank sees the same gathered report
    placement = S.place(queue, 4)
    expect = sorted((j.id, placement.devices[j.id][0]) for j in queue.jobs())
    assert r0[1] == expect                                 # each job ran once, on its placed device
    busy = r0[2]
    assert set(busy) == {0, 1, 2, 3}
    # two processes drive four devices: device busy clocks, a valid execution of the queue
    assert r0[4] == "device" and r0[3] == []
    assert r0[0] == pytest.approx(max(busy.values()))


def _wall_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(obj):
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    configs, queue, _ = _instance(n=8, G=2)
    rep = execute(queue, configs, 2, rank=rank, world=world, run_job=fake_run, all_gather=gather)
    tr = rep["trace"]
    out[rank] = (rep["clock"], rep["violations"], rep["makespan_s"], [(j.job_id, j.devices, j.start_s, j.end_s)
                                                                      for j in tr.jobs])
    dist.destroy_process_group()


def test_engine_wall_clock_one_process_per_gpu():
    """world == gpu_count: the makespan is the shared wall clock, the executed trace
    passes the feasibility re-check, and jobs on one device never overlap."""
    configs, queue, _ = _instance(n=8, G=2)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_wall_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    clock, violations, makespan, jobs = out[0]
    assert clock == "wall" and violations == []
    assert makespan == pytest.approx(max(e for _, _, _, e in jobs))
    assert sorted(j for j, *_ in jobs) == sorted(j.id for j in queue.jobs())


def test_check_feasibility_catches_bad_traces():
    from paper_2508_02932_b200.sweep.trace import ScheduleTrace, TraceJob, check_feasibility

    configs, queue, _ = _instance(n=6, G=2)
    jobs = queue.jobs()
    good = []
    t = {0: 0.0, 1: 0.0}
    for k, j in enumerate(jobs):
        devs = (0, 1) if j.degree == 2 else (k % 2,)
        s = max(t[d] for d in devs)
        good.append(TraceJob(j.id, j.configs, j.degree, s, 1.0, devs, j.predicted_time))
        for d in devs:
            t[d] = s + 1.0
    ok = ScheduleTrace(tuple(good), max(x.end_s for x in good), 2)
    assert check_feasibility(ok, queue) == []
    # two jobs on one device at the same time
    bad = list(good)
    bad[1] = TraceJob(jobs[1].id, jobs[1].configs, good[1].degree, good[0].start_s, 1.0, good[0].devices, 0.0)
    v = check_feasibility(ScheduleTrace(tuple(bad), max(x.end_s for x in bad), 2), queue)
    assert any("overlap on device(s)" in m for m in v)
    # a job missing, a device outside the pool, a wrong makespan
    v = check_feasibility(ScheduleTrace(tuple(good[1:]), 99.0, 2), queue)
    assert any("executed 0 times" in m for m in v) and any("makespan" in m for m in v)
    bad = list(good)
    bad[0] = TraceJob(jobs[0].id, jobs[0].configs, 1, 0.0, 1.0, (5,), 0.0)   # also the wrong device count
    assert any("outside the pool" in m for m in check_feasibility(ScheduleTrace(tuple(bad), ok.makespan, 2), queue))


def test_rank_schedule_matches_placement_and_covers_queue():
    configs, queue, _ = _instance(n=14, G=4)
    pl = S.place(queue, 4)
    seen = []
    for dev in range(4):
        sched = rank_schedule(queue, pl, dev)
        starts = [pl.start_s[j.id] for j in sched]
        assert starts == sorted(starts)
        seen += [j.id for j in sched]
    # a degree-d job appears in the schedule of each of its d devices
    assert sorted(seen) == sorted(j.id for j in queue.jobs() for _ in range(j.degree))


def test_profiles_calibrate_time_model():
    configs, queue, _ = _instance()
    rep = execute(queue, configs, 4, run_job=fake_run)
    assert len(rep["profiles"]) == len(queue.jobs())
    tm = S.calibrate_time_model(rep["profiles"] * 1 + [S.ProfileRecord(1, (8,), (1,), 16, 0.11)])
    assert tm.has_degree(1)


def _tp_instance(n=4, G=2):
    """Adapters too big for one GPU at degree 1 but fitting at degree 2 -> degree-2 (TP) jobs."""
    model = S.ModelSpec("m", 1, (S.TargetModule("q", 1 << 20, 1 << 20),), 0, 2)
    configs = [S.LoraConfig(f"t{i:02d}", rank=8, alpha=16.0, batch_size=1, learning_rate=1e-4, seq_len=16,
                            train_steps=2) for i in range(n)]
    per = S.lora_state_memory(configs[0], model, S.ShardingSpec()).total_bytes
    pool = S.GpuPool(G, int(per * 0.8))
    tm = S.TimeModel(coeffs={1: (1.0, 1e-4), 2: (0.5, 0.5e-4)})
    mem = S.MemoryContext(model, pool, configs)
    return configs, S.plan_jobs(G, configs, tm, mem)


def fake_run_tp(job, by_id, dev, tp=None):
    import torch
    assert tp is not None and tp.world == job.degree
    x = torch.tensor([float(tp.rank + 1)])
    tp.all_reduce_(x)                      # the job's own TP group
    return 1, 0.5, 0.5, [float(x.item())]


def _tp_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(obj):
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    configs, queue = _tp_instance()
    rep = execute(queue, configs, world, rank=rank, world=world, run_job=fake_run_tp, all_gather=gather)
    out[rank] = ([(r.job_id, r.device, r.losses) for r in rep["records"]], [p.parallelism_degree for p in rep["profiles"]])
    dist.destroy_process_group()


def test_engine_tensor_parallel_jobs_gloo():
    configs, queue = _tp_instance()
    assert queue.jobs() and all(j.degree == 2 for j in queue.jobs())
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_tp_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    recs, degrees = out[0]
    assert out[1][0] == recs
    # every TP job ran on both devices, and its all-reduce summed 1 + 2 over the job's group
    assert sorted((j, d) for j, d, _ in recs) == sorted((j.id, d) for j in queue.jobs() for d in (0, 1))
    assert all(loss == (3.0,) for _, _, loss in recs)
    assert degrees == [2] * len(queue.jobs())
