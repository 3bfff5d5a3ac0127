"""The execution engine running planner jobs of degree 2 as real tensor-parallel packed
training (PackedLoraTrainer shards, sequence parallel) -- two processes on one B200
over torch.distributed (gloo standing in for NCCL): every degree-2 job runs on both
ranks in its own process group and both ranks report the same losses."""

import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_02932_b200 import sweep as S
from paper_2508_02932_b200.sweep.engine import execute

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _instance(n=3, G=2):
    """Tiny-model configs whose adapter state only fits at degree 2 -> degree-2 (TP) jobs."""
    model = S.ModelSpec("m", 1, (S.TargetModule("q", 1 << 20, 1 << 20),), 0, 2)
    configs = [S.LoraConfig(f"e{i:02d}", rank=8, alpha=16.0 * (1 + i), batch_size=1,
                            learning_rate=1e-4 * (1 + i), seq_len=128, train_steps=2) for i in range(n)]
    per = S.lora_state_memory(configs[0], model, S.ShardingSpec()).total_bytes
    pool = S.GpuPool(G, int(per * 0.8))
    tm = S.TimeModel(coeffs={1: (1.0, 1e-4), 2: (0.5, 0.5e-4)})
    return configs, S.plan_jobs(G, configs, tm, S.MemoryContext(model, pool, configs))


def _worker(rank, world, port, ckpt, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def gather(obj):
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    configs, queue = _instance()
    rep = execute(queue, configs, world, rank=rank, world=world, model_name="tiny", steps_override=2,
                  all_gather=gather, checkpoint_dir=ckpt)
    out[rank] = sorted((r.job_id, r.device, r.losses) for r in rep["records"])
    dist.destroy_process_group()


def test_engine_runs_tensor_parallel_jobs_on_two_processes(tmp_path):
    configs, queue = _instance()
    assert queue.jobs() and all(j.degree == 2 for j in queue.jobs())
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), out), nprocs=2, join=True)
    recs = out[0]
    assert recs == out[1]
    jobs = {j.id: j for j in queue.jobs()}
    for jid in jobs:
        mine = [r for r in recs if r[0] == jid]
        assert sorted(d for _, d, _ in mine) == [0, 1]                 # both ranks of the TP group
        assert mine[0][2] == mine[1][2]                                 # identical (all-reduced) losses
        assert len(mine[0][2]) == len(jobs[jid].configs) and all(math.isfinite(x) for x in mine[0][2])
    # checkpoint pool: every configuration's adapter, gathered over its TP group, full size
    from paper_2508_02932_b200.checkpoint import load_adapter
    from paper_2508_02932_b200.model import PRESETS
    cfg = PRESETS["tiny"]
    for c in configs:
        state, meta = load_adapter(tmp_path / c.id)
        assert meta["degree"] == 2 and meta["r"] == c.rank
        shapes = {k: tuple(v.shape) for k, v in state.items()}
        assert shapes["base_model.model.model.layers.1.mlp.down_proj.lora_A.weight"] == (c.rank, cfg.ffn)
        assert shapes["base_model.model.model.layers.1.mlp.gate_proj.lora_B.weight"] == (cfg.ffn, c.rank)
        assert shapes["base_model.model.model.layers.0.self_attn.q_proj.lora_B.weight"] == (cfg.d, c.rank)
