"""Model-level parity at the BENCH SHAPES (config C3, Llama-3.1-8B: d = 4096, ffn = 14336,
32/8 heads, vocab 128256) at reduced depth and tokens, with the bench's own adapter
init (A ~ U(+-1/sqrt(h_in)), B ~ N(0, 0.02^2), alpha = r * {0.25, 1, 2, 4}, ranks
8/16/32/64): the packed trainer vs the fp64 oracle decoder whose every LoRA linear is
the reference's packed_forward / packed_backward restated (oracle/model_oracle.py).

Two layers, four adapters, one 256-token sequence each (T = 1024).  Tolerances are the
C1 tier of test_gpu_model.py: per-adapter loss |d|/|ref| <= 1e-2; LoRA gradients
pooled relative Frobenius <= 2e-2 and per (layer, target, factor, adapter) block
<= 5e-2 (blocks of the alpha = r/4 adapters carry the smallest gradients)."""

import dataclasses

import pytest
import torch

from oracle.model_oracle import from_trainer, oracle_step
from paper_2508_02932_b200.model import PRESETS, AdapterSpec, PackedLoraTrainer

pytestmark = pytest.mark.gpu


def test_c3_shapes_two_layers_match_oracle():
    cfg = dataclasses.replace(PRESETS["llama-3.1-8b"], n_layers=2)
    s = 256
    mults, lrs = [0.25, 1.0, 2.0, 4.0], [2e-5, 5e-5, 1e-4, 2e-4]
    specs = [AdapterSpec(rank=r, alpha=r * m, batch=1, lr=lr) for r, m, lr in zip((8, 16, 32, 64), mults, lrs)]
    tr = PackedLoraTrainer(cfg, specs, s, device="cuda")          # bench init (b_std 0.02, a ~ U(1/sqrt(h_in)))
    tokens = tr.synthetic_tokens().cuda()
    losses = tr.forward_backward(tokens).double().cpu()
    base, adapters = from_trainer(tr)
    ref_losses, ref_grads, _ = oracle_step(cfg, base, adapters, [sp.alpha for sp in specs], tr.meta.row_offsets,
                                           tokens.cpu(), s, tr.cos.double().cpu(), tr.sin.double().cpu(),
                                           [sp.batch * (s - 1) for sp in specs])
    rel = ((losses - ref_losses).abs() / ref_losses.abs()).max().item()
    num = den = worst = 0.0
    for (layer, tname), (dd, du) in ref_grads.items():
        for i, sp in enumerate(specs):
            ga = tr.bank.block(tr.bank.G, layer, tname, "A", i)[:, :sp.rank].double().cpu()
            gb = tr.bank.block(tr.bank.G, layer, tname, "B", i)[:, :sp.rank].double().cpu().t()
            for got, ref in ((ga, dd[i]), (gb, du[i])):
                e, rn = (got - ref).norm().item(), ref.norm().item()
                num, den = num + e * e, den + rn * rn
                worst = max(worst, e / max(rn, 1e-30))
    pooled = (num / den) ** 0.5
    print(f"C3 shapes, 2 layers: loss rel err {rel:.3e} ({losses.tolist()} vs {ref_losses.tolist()}); "
          f"grads worst block {worst:.3e}, pooled {pooled:.3e}")
    assert rel <= 1e-2
    assert pooled <= 2e-2
    assert worst <= 5e-2
