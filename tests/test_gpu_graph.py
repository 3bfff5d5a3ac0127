"""model.GraphedStep: the packed training step captured as one CUDA graph and replayed
must train exactly like the eager step (same kernels, same order; per-adapter AdamW step
counts on the device), and count its libplora launches."""

import pytest
import torch

from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

pytestmark = pytest.mark.gpu


def _make(preset):
    specs, s = bench_adapters(preset)
    return PackedLoraTrainer(PRESETS[preset], specs, s, device="cuda", a_scale=0.05,
                             b_std=[0.2 / x.alpha for x in specs])


@pytest.mark.parametrize("preset", ["tiny", "tiny-qwen"])
def test_graphed_step_trains_like_eager(preset):
    eager, graphed_tr = _make(preset), _make(preset)
    tokens = eager.synthetic_tokens().cuda()
    other = eager.synthetic_tokens(seed_base=7).cuda()
    # eager: 2 warm-up steps (what GraphedStep runs before capture), then 3 steps alternating batches
    ref = []
    for t in (tokens, tokens, tokens, other, tokens):
        ref.append(eager.step(t).clone())
    g = graphed_tr.graphed(tokens, warmup=2)
    got = []
    l0 = ops.launch_count()
    for t in (tokens, other, tokens):
        got.append(g.step(t).clone())
    assert ops.launch_count() - l0 == 3 * g.launches_per_step > 0
    torch.cuda.synchronize()
    for a, b in zip(ref[2:], got):
        assert torch.allclose(a, b, rtol=1e-3, atol=1e-5), (a, b)
    assert torch.allclose(eager.bank.P, graphed_tr.bank.P, rtol=1e-3, atol=1e-6)
    assert torch.equal(eager.bank.hp[:, 2], graphed_tr.bank.hp[:, 2])          # 5 optimizer steps each
    assert graphed_tr.bank.step_count == eager.bank.step_count == 5
