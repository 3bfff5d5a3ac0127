"""ops.PackedLoraLinear -- the torch autograd op over plora_linear_fwd / plora_linear_bwd --
against the oracle (the reference's packed_forward / packed_backward restated in fp64,
oracle/lorapack_oracle.py) at the bf16 tier: rel-Frobenius <= 1e-2 and max|err|/max|ref|
<= 2e-2 per adapter; and a torch optimizer step through the op."""

import numpy as np
import pytest
import torch

from oracle import lorapack_oracle as O
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta

pytestmark = pytest.mark.gpu

REL_FROB = 1e-2
MAX_REL = 2e-2


def _close(got, ref, what):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    assert got.shape == ref.shape, what
    rf, mr = O.rel_frobenius(got, ref), O.max_abs_over_max_ref(got, ref)
    assert rf <= REL_FROB and mr <= MAX_REL, f"{what}: rel_frob={rf:.3e} max_rel={mr:.3e}"


@pytest.mark.parametrize("ranks,tokens,d,k", [
    ((8, 16, 32, 64), (256, 128, 384, 130), 256, 512),
    ((4, 70, 12), (64, 300, 1), 192, 320),          # rank > 64 (two rank blocks), ragged and tiny segments
    ((16,) * 3, (2048, 1024, 1024), 1024, 1024),
])
def test_packed_lora_linear_matches_oracle(ranks, tokens, d, k):
    torch.manual_seed(0)
    dev = torch.device("cuda", 0)
    alphas = [0.5 * r for r in ranks]
    meta = build_meta(list(ranks), list(tokens), alphas)
    w = (torch.randn(k, d, device=dev) * 0.05).to(torch.bfloat16)          # nn.Linear layout [k][d]
    lin = ops.PackedLoraLinear(meta, w, init_std=0.05, seed=3)
    T = sum(tokens)
    x = torch.randn(T, d, device=dev).to(torch.bfloat16).requires_grad_()
    y = lin(x)
    dy = torch.randn(T, k, device=dev).to(torch.bfloat16)
    y.backward(dy)

    # oracle on the same (bf16-valued) operands, fp64
    so = meta.row_offsets
    X = x.detach().double().cpu().numpy()
    W = w.double().cpu().numpy().T                        # reference layout [d][k]
    downs = [lin.down(i).detach().to(torch.bfloat16).double().cpu().numpy() for i in range(len(ranks))]
    ups = [lin.up(i).detach().to(torch.bfloat16).double().cpu().numpy() for i in range(len(ranks))]
    xs = [X[so[i]:so[i + 1]] for i in range(len(ranks))]
    p = O.pack(downs, ups, alphas, xs)
    ref_y = np.concatenate(O.packed_forward(p, W))
    _close(y.detach().double().cpu().numpy(), ref_y, "y")
    dys = [dy.double().cpu().numpy()[so[i]:so[i + 1]] for i in range(len(ranks))]
    rd, ru, rx = O.packed_backward(p, W, dys)
    _close(x.grad.double().cpu().numpy(), np.concatenate(rx), "dx")
    ga, gb = lin.a.grad, lin.b.grad
    ro = meta.rpad_off
    for i, r in enumerate(ranks):
        blk_a = ga[d * int(ro[i]): d * int(ro[i + 1])].view(d, -1)
        blk_b = gb[k * int(ro[i]): k * int(ro[i + 1])].view(k, -1)
        _close(blk_a[:, :r].double().cpu().numpy(), rd[i], f"dA[{i}]")
        _close(blk_b[:, :r].t().double().cpu().numpy(), ru[i], f"dB[{i}]")
        if blk_a.shape[1] > r:   # padding columns of the region carry exactly zero gradient
            assert float(blk_a[:, r:].abs().max()) == 0.0 and float(blk_b[:, r:].abs().max()) == 0.0


def test_packed_lora_linear_optimizer_step_refreshes_shadows():
    """A torch optimizer updates the fp32 masters; the next forward sees them (bf16 shadows
    refreshed from the new parameter versions)."""
    dev = torch.device("cuda", 0)
    meta = build_meta([8, 16], [128, 256], [16.0, 8.0])
    w = (torch.randn(256, 128, device=dev) * 0.05).to(torch.bfloat16)
    lin = ops.PackedLoraLinear(meta, w, init_std=0.05)
    x = torch.randn(384, 128, device=dev).to(torch.bfloat16)
    opt = torch.optim.AdamW(lin.parameters(), lr=1e-2)
    y0 = lin(x)
    (y0.float() ** 2).mean().backward()
    opt.step()
    y1 = lin(x)
    assert lin.a_sh[0, :, :8].float().sub(lin.down(0).float()).abs().max() < 1e-2
    assert not torch.equal(y0, y1)
    # the same op with the updated masters loaded into a fresh module gives the same output
    lin2 = ops.PackedLoraLinear(meta, w)
    with torch.no_grad():
        lin2.a.copy_(lin.a)
        lin2.b.copy_(lin.b)
    assert torch.equal(lin2(x), y1)
