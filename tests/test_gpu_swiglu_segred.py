"""SwiGLU backward fused with the down projection's dA (ops.swiglu_bwd_segred /
plora_swiglu_bwd_segred) against the two-kernel path it replaces (plora_swiglu_bwd with the
activation re-emitted, then the K5 segment reduction over it): dg, du and dA bit-identical;
and dA against a torch fp32 restatement of the reference's Case 3 (lorapack.py:226) on
act = silu(g) u.  Packs with segments that are not multiples of 64 tokens (direct-store
tail k-blocks), an empty segment, ffn not a multiple of 128 (partial column tile), the C3
shape, in place (dg / du over g / u) and out of place."""

import pytest
import torch

from paper_2508_02932_b200 import elementwise as ew
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta

pytestmark = pytest.mark.gpu

bf = torch.bfloat16

CASES = [
    ("c3", [8, 16, 32, 64] * 4, [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]], 14336),
    ("ragged", [8, 64, 16, 32, 8, 64, 1, 48], [4096, 1024, 0, 2048, 333, 1024, 100, 1500], 1792),
    ("narrow", [16, 64], [130, 700], 200),   # ffn % 128 != 0, short segments
]


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


def _operands(ranks, tokens, ffn, seed):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    meta = build_meta(ranks, tokens, [1.0] * len(ranks)).to("cuda")
    T = meta.total_tokens
    da = (torch.randn(T, ffn, device="cuda", generator=gen) * 0.1).to(bf)
    g = (torch.randn(T, ffn, device="cuda", generator=gen) * 2).to(bf)
    u = torch.randn(T, ffn, device="cuda", generator=gen).to(bf)
    dh = torch.zeros(T, meta.rpad64, device="cuda", dtype=bf)
    for i, r in enumerate(ranks):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        dh[s:e, :r] = (torch.randn(e - s, r, device="cuda", generator=gen) * 0.1).to(bf)
    return meta, da, g, u, dh


@pytest.mark.parametrize("name,ranks,tokens,ffn", CASES)
@pytest.mark.parametrize("inplace", [True, False])
def test_fused_equals_two_kernels(name, ranks, tokens, ffn, inplace):
    meta, da, g, u, dh = _operands(ranks, tokens, ffn, seed=7)
    T = meta.total_tokens
    # two-kernel reference path
    act = torch.empty_like(g)
    dg_ref, du_ref = ew.swiglu_bwd(da, g, u, act_out=act)
    ga_ref = torch.full((ffn * meta.rpad16_total,), float("nan"), device="cuda")
    ops.segred(meta, act, dh, ga_ref)
    # fused
    ga = torch.full_like(ga_ref, float("nan"))
    g2, u2 = g.clone(), u.clone()
    if inplace:
        dg, du = ops.swiglu_bwd_segred(meta, da, g2, u2, dh, ga, out_g=g2, out_u=u2)
        assert dg.data_ptr() == g2.data_ptr() and du.data_ptr() == u2.data_ptr()
    else:
        dg, du = ops.swiglu_bwd_segred(meta, da, g2, u2, dh, ga)
        assert torch.equal(g2, g) and torch.equal(u2, u)     # inputs untouched
    torch.cuda.synchronize()
    assert torch.equal(dg, dg_ref) and torch.equal(du, du_ref)
    assert not torch.isnan(ga).any()
    if len(ranks) * ((ffn + 127) // 128) * 4 <= torch.cuda.get_device_properties(0).multi_processor_count:
        # packs this small run the separate K5 as stream-K (other fp32 association)
        assert rel(ga, ga_ref) < 1e-6
    else:   # same LPT tiles, same MMA order
        assert torch.equal(ga, ga_ref)
    for i, r in enumerate(ranks):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk = ga[ffn * int(meta.rpad_off[i]): ffn * int(meta.rpad_off[i + 1])].view(ffn, rp)
        if e == s:
            assert not torch.any(blk)
            continue
        a32 = torch.nn.functional.silu(g[s:e].float()) * u[s:e].float()
        ref = a32.to(bf).float().t() @ dh[s:e, :rp].float()        # Case 3 on the bf16 activation
        assert rel(blk, ref) < 1e-4, (name, i)


def test_trainer_fused_swiglu_bwd_matches():
    """A C1-shaped step with and without the fusion: identical losses and gradients."""
    from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

    specs, s = bench_adapters("tiny")
    res = []
    for fuse in (True, False):
        tr = PackedLoraTrainer(PRESETS["tiny"], specs, s, device="cuda", a_scale=0.05, b_std=0.05,
                               fuse_swiglu_bwd=fuse)
        tokens = tr.synthetic_tokens().cuda()
        losses = tr.forward_backward(tokens).float().clone()
        res.append((losses, tr.bank.G.clone()))
    assert torch.equal(res[0][0], res[1][0])
    assert torch.equal(res[0][1], res[1][1])


def test_round_robin_tiles_without_host_offsets():
    """A pack without host row offsets (plora_pack_t.h_row_off = NULL) runs the tiles
    round-robin instead of the LPT schedule: same tiles, same MMA order, bit-identical."""
    meta, da, g, u, dh = _operands(*CASES[1][1:3], 1792, seed=9)
    ga = torch.empty(1792 * meta.rpad16_total, device="cuda")
    dg, du = ops.swiglu_bwd_segred(meta, da, g, u, dh, ga)
    saved = meta.struct.h_row_off
    meta.struct.h_row_off = None
    try:
        ga2 = torch.full_like(ga, float("nan"))
        dg2, du2 = ops.swiglu_bwd_segred(meta, da, g, u, dh, ga2)
    finally:
        meta.struct.h_row_off = saved
    torch.cuda.synchronize()
    assert torch.equal(dg, dg2) and torch.equal(du, du2) and torch.equal(ga, ga2)
