"""Tensor-parallel packed LoRA (config C4's path) on ONE B200: a TP group of g ranks
runs as g threads sharing the GPU (tp.ThreadComm, each rank on its own stream, the
same sharded kernels and all-reduce placement the NCCL path uses).  The sharded
job is compared directly with the fp64 oracle decoder (oracle/model_oracle.py: every
LoRA linear is the reference's packed_forward / packed_backward restated), on the
unsharded model's weights, at the C1 tier of test_gpu_model.py:

  per-adapter loss                     |d| / |ref| <= 1e-2
  per-(layer, target, factor, adapter) gradient, shards reassembled:
                                       relative Frobenius <= 3e-2 (pooled <= 2e-2)
  replicated factors (column A, row B) bit-identical on every rank, before and
  after a fused AdamW step (no gradient all-reduce is needed for them)."""

import pytest
import torch

from oracle.model_oracle import from_trainer, oracle_step
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters
from paper_2508_02932_b200.tp import TPShard, run_threaded

pytestmark = pytest.mark.gpu


def _make(preset, tp=None, sp=True, save_normed=None, fused=False):
    cfg = PRESETS[preset]
    specs, s = bench_adapters(preset)
    return PackedLoraTrainer(cfg, specs, s, device="cuda", a_scale=0.05, b_std=[0.2 / x.alpha for x in specs],
                             tp=tp, sequence_parallel=sp, save_normed=save_normed, tp_fused=fused)


def _grads(tr):
    out = {}
    bank = tr.bank
    for layer in range(tr.cfg.n_layers):
        for t in bank.targets:
            for kind in ("A", "B"):
                for i in range(tr.meta.n_adapters):
                    r = tr.meta.ranks[i]
                    out[(layer, t.name, kind, i)] = bank.block(bank.G, layer, t.name, kind, i)[:, :r].float().cpu()
    return out


def oracle_reference(tr, tokens):
    """fp64 oracle losses and per-(layer, target, factor, adapter) LoRA gradients of the
    unsharded model ``tr`` (its weights only: nothing of ``tr`` runs), keyed and laid out
    like _grads (A_i [h_in][r], B_i^T [h_out][r])."""
    base, adapters = from_trainer(tr)
    n_lab = [sp.batch * (tr.s - 1) for sp in tr.specs]
    losses, grads, _ = oracle_step(tr.cfg, base, adapters, [sp.alpha for sp in tr.specs], tr.meta.row_offsets,
                                   tokens.cpu(), tr.s, tr.cos.double().cpu(), tr.sin.double().cpu(), n_lab)
    out = {}
    for (layer, tname), (dd, du) in grads.items():
        for i in range(tr.meta.n_adapters):
            out[(layer, tname, "A", i)] = dd[i].float()
            out[(layer, tname, "B", i)] = du[i].t().float()
    return losses.double(), out


def _masters(tr):
    bank = tr.bank
    return {(layer, t.name, kind, i): bank.block(bank.P, layer, t.name, kind, i).cpu().clone()
            for layer in range(tr.cfg.n_layers) for t in bank.targets for kind in ("A", "B")
            for i in range(tr.meta.n_adapters)}


@pytest.mark.parametrize("preset,g,sp,keep,fused", [("tiny-qwen", 2, True, True, False), ("tiny", 4, True, True, False),
                                                    ("tiny-qwen", 2, True, False, False),
                                                    ("tiny-qwen", 2, False, True, False),
                                                    ("tiny", 4, False, True, False), ("tiny-qwen", 2, True, True, True)])
def test_tp_matches_oracle(preset, g, sp, keep, fused):
    """sp: Megatron sequence parallelism (token-sharded residual stream; g = 2 cuts the
    pair-tile list exactly at the shard boundaries -> per-shard reduces overlapping the
    GEMM; g = 4 does not -> one reduce-scatter); sp = False: all-reduce chunks.
    keep = False: the normed inputs are re-gathered in the backward on the side stream.
    fused: the row-parallel GEMMs reduce their tiles straight into the owning rank's
    buffer (TMA reduce-add into peer memory -- here the other threads' buffers)."""
    ref = _make(preset)                      # unsharded weights for the oracle (not run)
    tokens = ref.synthetic_tokens().cuda()
    ref_losses, ref_grads = oracle_reference(ref, tokens)
    del ref

    def rank_fn(comm):
        tr = _make(preset, tp=comm, sp=sp, save_normed=keep, fused=fused)
        assert tr.sp == sp and tr.tp_fused == fused
        losses = tr.forward_backward(tokens).double().cpu()
        grads = _grads(tr)
        tr.bank.adamw_step()
        torch.cuda.current_stream().synchronize()
        return losses, grads, _masters(tr)

    outs = run_threaded(g, rank_fn)
    for losses, _, _ in outs:
        rel = ((losses - ref_losses).abs() / ref_losses.abs()).max().item()
        assert rel <= 1e-2, (rel, losses, ref_losses)
    # every rank computes identical losses (all-reduced CE statistics)
    for losses, _, _ in outs[1:]:
        assert torch.equal(losses, outs[0][0])

    num = den = worst = 0.0
    for key, want in ref_grads.items():
        layer, tname, kind, i = key
        sh = TPShard(0, g)
        if sh.replicated(tname, kind):
            got = outs[0][1][key]
            for r in range(1, g):
                assert torch.equal(outs[r][1][key], got), key      # bit-identical replicas
                assert torch.equal(outs[r][2][key], outs[0][2][key]), key
        else:
            got = torch.cat([outs[r][1][key] for r in range(g)], 0)
        assert got.shape == want.shape, (key, got.shape, want.shape)
        e = (got - want).norm().item()
        rn = want.norm().item()
        num += e * e
        den += rn * rn
        worst = max(worst, e / max(rn, 1e-30))
    print(f"tp={g} sp={sp} fused={fused} {preset}: worst per-block grad rel-Frob {worst:.3e}, pooled {(num / den) ** 0.5:.3e}")
    assert worst <= 3e-2
    assert (num / den) ** 0.5 <= 2e-2


def test_tp_shards_are_slices_of_unsharded_model():
    """Sharded base weights / adapter masters are exact slices of the unsharded ones."""
    ref = _make("tiny-qwen")

    def rank_fn(comm):
        tr = _make("tiny-qwen", tp=comm)
        torch.cuda.current_stream().synchronize()
        return tr

    trs = run_threaded(2, rank_fn)
    cfg = ref.cfg
    for r, tr in enumerate(trs):
        sh = TPShard(r, 2)
        for layer in range(cfg.n_layers):
            for t in cfg.targets():
                rows, cols = sh.weight_slice(t.name, t.h_in, t.h_out)
                assert torch.equal(tr.base.layers[layer][t.name], ref.base.layers[layer][t.name][rows, cols])
                for kind in ("A", "B"):
                    for i in range(ref.meta.n_adapters):
                        sl = sh.lora_rows(t.name, kind, t.h_in, t.h_out)
                        assert torch.equal(tr.bank.block(tr.bank.P, layer, t.name, kind, i),
                                           ref.bank.block(ref.bank.P, layer, t.name, kind, i)[sl])
        assert torch.equal(tr.base.lm_head, ref.base.lm_head[sh.span(cfg.vocab)])


def test_abi_nccl_comm_single_rank():
    """The C-ABI TP collectives (plora_tp_comm_init / allreduce / allgather / reducescatter /
    reduce over NCCL) on a one-rank group: all are the identity, bf16 and f32."""
    from paper_2508_02932_b200.tp import AbiNcclComm
    comm = AbiNcclComm()
    try:
        for dt in (torch.bfloat16, torch.float32):
            x = torch.randn(4097, device="cuda").to(dt)
            y = x.clone()
            comm.all_reduce_(y)
            comm.all_reduce_(y, "max")
            comm.reduce_(y, 0)
            g = torch.empty_like(y)
            comm.all_gather_(g, y)
            r = torch.empty_like(y)
            comm.reduce_scatter_(r, g)
            torch.cuda.synchronize()
            assert torch.equal(x, y) and torch.equal(x, g) and torch.equal(x, r)
    finally:
        comm.close()


def test_tp_checkpoint_gathers_full_adapters():
    """checkpoint.adapter_state on a TP group (collective all-gather of the sharded
    factors) == the unsharded trainer's adapter, exactly."""
    from paper_2508_02932_b200.checkpoint import adapter_state
    ref = _make("tiny-qwen")
    want = [adapter_state(ref, i) for i in range(ref.meta.n_adapters)]

    def rank_fn(comm):
        tr = _make("tiny-qwen", tp=comm)
        return [adapter_state(tr, i) for i in range(tr.meta.n_adapters)]

    for states in run_threaded(2, rank_fn):
        for got, exp in zip(states, want):
            assert got.keys() == exp.keys()
            for k in exp:
                assert torch.equal(got[k], exp[k]), k
