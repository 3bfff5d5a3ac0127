"""Tensor + sequence parallel packed trainer as TWO PROCESSES on one B200, talking
through torch.distributed (tp.DistComm) -- the code path a real TP job uses, with the
gloo backend standing in for NCCL (NCCL refuses two ranks on one device; gloo moves
CUDA tensors through the host).  Each rank builds its Megatron shard, runs one
forward + backward and a fused AdamW step; the parent compares with the fp64 oracle
decoder on the unsharded model's weights (same tolerances as test_gpu_tp.py) and
checks the replicated factors are bit-identical across the two processes."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters
from paper_2508_02932_b200.tp import DistComm, TPShard
from tests.test_gpu_tp import oracle_reference

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _make(tp=None, save_normed=None, fused=False):
    cfg = PRESETS["tiny-qwen"]
    specs, s = bench_adapters("tiny-qwen")
    return PackedLoraTrainer(cfg, specs, s, device="cuda", a_scale=0.05, b_std=[0.2 / x.alpha for x in specs],
                             tp=tp, save_normed=save_normed, tp_fused=fused)


def _grads(tr):
    bank = tr.bank
    return {(layer, t.name, kind, i): bank.block(bank.G, layer, t.name, kind, i)[:, :tr.meta.ranks[i]].float().cpu()
            for layer in range(tr.cfg.n_layers) for t in bank.targets for kind in ("A", "B")
            for i in range(tr.meta.n_adapters)}


def _worker(rank, world, port, keep, fused, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tr = _make(DistComm(), save_normed=keep, fused=fused)
    assert tr.sp and tr.tp_fused == fused
    tokens = tr.synthetic_tokens().cuda()
    losses = tr.forward_backward(tokens).double().cpu()
    grads = _grads(tr)
    tr.bank.adamw_step()
    torch.cuda.synchronize()
    masters = {k: tr.bank.block(tr.bank.P, *k).cpu().clone() for k in grads}
    out[rank] = (losses, grads, masters)
    dist.destroy_process_group()


@pytest.mark.parametrize("keep,fused", [(True, False), (False, False)])
def test_tp2_two_processes_gloo(keep, fused):
    """(The fused peer-memory path is not covered here: torch symmetric memory refuses two
    ranks on one device -- "allocations from overlapping devices"; test_gpu_tp.py covers
    it with thread-emulated ranks.)"""
    ref = _make()                            # unsharded weights for the oracle (not run)
    tokens = ref.synthetic_tokens().cuda()
    ref_losses, ref_grads = oracle_reference(ref, tokens)
    del ref
    torch.cuda.empty_cache()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), keep, fused, out), nprocs=2, join=True)
    (l0, g0, m0), (l1, g1, m1) = out[0], out[1]
    assert torch.equal(l0, l1)
    assert ((l0 - ref_losses).abs() / ref_losses.abs()).max().item() <= 1e-2
    num = den = worst = 0.0
    for key, want in ref_grads.items():
        _, tname, kind, _ = key
        if TPShard(0, 2).replicated(tname, kind):
            assert torch.equal(g0[key], g1[key]) and torch.equal(m0[key], m1[key]), key
            got = g0[key]
        else:
            got = torch.cat([g0[key], g1[key]], 0)
        e = (got - want).norm().item()
        rn = want.norm().item()
        num += e * e
        den += rn * rn
        worst = max(worst, e / max(rn, 1e-30))
    assert worst <= 3e-2
    assert (num / den) ** 0.5 <= 2e-2
