"""Model-level parity at config C1 (tiny d=256, 2 layers, 4 adapters r=8/16/32/64):
the B200 packed trainer vs the fp64 oracle decoder whose every LoRA linear is the
oracle restatement of lorasweep.packed_forward/packed_backward.

Tolerance tier (bf16 activations end to end, fp32 accumulation / fp32 grads):
  per-adapter loss   |d| / |ref| <= 1e-2
  per-(layer, target, adapter) LoRA gradient: relative Frobenius <= 3e-2
  (all gradients pooled: relative Frobenius <= 2e-2)"""

import numpy as np
import pytest
import torch

from oracle import lorapack_oracle as O
from oracle.model_oracle import from_trainer, oracle_step
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

pytestmark = pytest.mark.gpu


def _trainer(specs=None, seeds=None, preset="tiny"):
    """C1 with the bench ranks/alphas (alpha = r * {0.25,1,2,4} up to 256).  B_i is drawn
    with std 0.2/alpha_i so every adapter's low-rank term is O(1) next to the base path:
    with B ~ N(0, 0.05^2) the alpha=256 adapter's term is ~100x the base output, the
    random-weight network saturates its attention and the bf16-vs-fp64 comparison
    measures chaos, not the kernels."""
    cfg = PRESETS[preset]
    sp, s = bench_adapters(preset)
    specs = specs or sp
    return PackedLoraTrainer(cfg, specs, s, device="cuda", adapter_seeds=seeds, a_scale=0.05,
                             b_std=[0.2 / x.alpha for x in specs])


def _oracle(tr, tokens):
    base, adapters = from_trainer(tr)
    n_lab = [sp.batch * (tr.s - 1) for sp in tr.specs]
    cos, sin = tr.cos.double().cpu(), tr.sin.double().cpu()
    return oracle_step(tr.cfg, base, adapters, [sp.alpha for sp in tr.specs], tr.meta.row_offsets,
                       tokens.cpu(), tr.s, cos, sin, n_lab)


@pytest.mark.parametrize("preset", ["tiny", "tiny-qwen"])
def test_tiny_model_matches_oracle(preset):
    """tiny = C1 (Llama-style); tiny-qwen = the same size with C2/C4's Qwen2 features
    (GQA 4/2, q/k/v bias, tied embeddings)."""
    tr = _trainer(preset=preset)
    tokens = tr.synthetic_tokens().cuda()
    losses = tr.forward_backward(tokens).cpu().double()
    ref_losses, ref_grads, _ = _oracle(tr, tokens)
    rel = ((losses - ref_losses).abs() / ref_losses.abs()).max().item()
    print("loss rel err", rel, losses.tolist(), ref_losses.tolist())
    assert rel <= 1e-2
    num = den = 0.0
    worst = 0.0
    n = tr.meta.n_adapters
    for (layer, tname), (dd, du) in ref_grads.items():
        for i in range(n):
            r = tr.meta.ranks[i]
            ga = tr.bank.block(tr.bank.G, layer, tname, "A", i)[:, :r].double().cpu()
            gb = tr.bank.block(tr.bank.G, layer, tname, "B", i)[:, :r].double().cpu().t()
            for got, ref in ((ga, dd[i]), (gb, du[i])):
                e = (got - ref).norm().item()
                rn = ref.norm().item()
                num += e * e
                den += rn * rn
                worst = max(worst, e / max(rn, 1e-30))
    print("worst per-block grad rel-Frob", worst, "pooled", (num / den) ** 0.5)
    assert worst <= 3e-2
    assert (num / den) ** 0.5 <= 2e-2


def test_padding_columns_stay_zero_after_steps():
    tr = _trainer()
    tokens = tr.synthetic_tokens().cuda()
    for _ in range(3):
        tr.step(tokens)
    m = tr.meta
    for (layer, tname, kind) in list(tr.bank.regions)[:6]:
        for i in range(m.n_adapters):
            blk = tr.bank.block(tr.bank.P, layer, tname, kind, i)
            assert not torch.any(blk[:, m.ranks[i]:])
            sh = tr.bank.shadow_of(layer, tname, kind)[i]
            assert torch.equal(sh[:, : blk.shape[1]].float(), blk.to(torch.bfloat16).float())


def test_loss_decreases_per_adapter():
    tr = _trainer()
    tokens = tr.synthetic_tokens().cuda()
    first = tr.step(tokens).clone()
    for _ in range(20):
        last = tr.step(tokens).clone()
    assert torch.all(last < first), (first.tolist(), last.tolist())


def test_packing_invariance_model_level():
    """Adapter i trained inside the pack == adapter i trained alone."""
    cfg_specs, s = bench_adapters("tiny")
    packed = _trainer()
    tokens = packed.synthetic_tokens().cuda()
    lp = packed.forward_backward(tokens).clone()
    i = 2
    solo = PackedLoraTrainer(PRESETS["tiny"], [cfg_specs[i]], s, device="cuda", base=packed.base,
                             adapter_seeds=[100 + i], a_scale=0.05, b_std=[0.2 / cfg_specs[i].alpha])
    ro = packed.meta.row_offsets
    ls = solo.forward_backward(tokens[ro[i]:ro[i + 1]].contiguous())
    assert abs(ls[0].item() - lp[i].item()) <= 1e-3 * abs(lp[i].item())
    for layer in range(2):
        for t in ("q", "down"):
            a = packed.bank.block(packed.bank.G, layer, t, "A", i)
            b = solo.bank.block(solo.bank.G, layer, t, "A", 0)
            assert O.rel_frobenius(b.cpu().numpy(), a.cpu().numpy()) <= 1e-2


def test_saved_and_recomputed_norms_bit_identical():
    """Keeping the normed inputs x1/x2 from the forward (save_normed) and recomputing
    them from (h, rstd) in the backward give bit-identical losses and gradients."""
    cfg = PRESETS["tiny"]
    sp, s = bench_adapters("tiny")
    kw = dict(device="cuda", a_scale=0.05, b_std=[0.2 / x.alpha for x in sp])
    a = PackedLoraTrainer(cfg, sp, s, save_normed=True, **kw)
    b = PackedLoraTrainer(cfg, sp, s, save_normed=False, base=a.base, **kw)
    tokens = a.synthetic_tokens().cuda()
    la = a.forward_backward(tokens).clone()
    lb = b.forward_backward(tokens).clone()
    assert torch.equal(la, lb)
    assert torch.equal(a.bank.G, b.bank.G)


def test_model_with_rank_above_64_matches_oracle():
    """An adapter of rank 96 (two 64-column rank blocks in every shadow / Hs / dH) next to
    small ranks, through the whole trainer, against the fp64 oracle decoder."""
    from paper_2508_02932_b200.model import AdapterSpec
    specs = [AdapterSpec(rank=96, alpha=48.0, batch=1, lr=1e-4), AdapterSpec(rank=8, alpha=16.0, batch=2, lr=2e-4),
             AdapterSpec(rank=40, alpha=10.0, batch=1, lr=5e-5)]
    tr = _trainer(specs=specs)
    assert tr.meta.nb == 2
    tokens = tr.synthetic_tokens().cuda()
    losses = tr.forward_backward(tokens).cpu().double()
    ref_losses, ref_grads, _ = _oracle(tr, tokens)
    assert ((losses - ref_losses).abs() / ref_losses.abs()).max().item() <= 1e-2
    num = den = 0.0
    for (layer, tname), (dd, du) in ref_grads.items():
        for i in range(tr.meta.n_adapters):
            r = tr.meta.ranks[i]
            ga = tr.bank.block(tr.bank.G, layer, tname, "A", i)[:, :r].double().cpu()
            gb = tr.bank.block(tr.bank.G, layer, tname, "B", i)[:, :r].double().cpu().t()
            for got, ref in ((ga, dd[i]), (gb, du[i])):
                num += (got - ref).norm().item() ** 2
                den += ref.norm().item() ** 2
    assert (num / den) ** 0.5 <= 2e-2
