"""Fused elementwise kernels (csrc/elementwise.cu) vs their torch fp32 restatements."""

import pytest
import torch

from paper_2508_02932_b200 import elementwise as ew

pytestmark = pytest.mark.gpu
bf = torch.bfloat16


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


@pytest.mark.parametrize("d", [256, 2048, 4096, 5120])
def test_rmsnorm(d):
    x = (torch.randn(300, d, device="cuda") * 3).to(bf)
    w = (torch.rand(d, device="cuda") + 0.5).to(bf)
    y, r = ew.rmsnorm_fwd(x, w, 1e-5)
    ry, rr = ew.ref_rmsnorm_fwd(x, w, 1e-5)
    assert rel(y, ry) < 4e-3 and torch.allclose(r, rr, rtol=1e-5)
    assert torch.equal(ew.rmsnorm_apply(x, r, w), y)
    dy = torch.randn(300, d, device="cuda").to(bf)
    res = torch.randn(300, d, device="cuda").to(bf)
    assert rel(ew.rmsnorm_bwd(dy, x, r, w), ew.ref_rmsnorm_bwd(dy, x, r, w)) < 4e-3
    assert rel(ew.rmsnorm_bwd(dy, x, r, w, res), ew.ref_rmsnorm_bwd(dy, x, r, w, res)) < 4e-3
    inplace = dy.clone()
    ew.rmsnorm_bwd(inplace, x, r, w, res, out=inplace)
    assert torch.equal(inplace, ew.rmsnorm_bwd(dy, x, r, w, res))


def test_add_rmsnorm():
    a = (torch.randn(257, 4096, device="cuda") * 2).to(bf)
    b = torch.randn(257, 4096, device="cuda").to(bf)
    w = (torch.rand(4096, device="cuda") + 0.5).to(bf)
    s_, y, r = ew.add_rmsnorm_fwd(a, b, w, 1e-5)
    ref_s = (a.float() + b.float()).to(bf)
    assert torch.equal(s_, ref_s)
    ry, rr = ew.ref_rmsnorm_fwd(ref_s, w, 1e-5)
    assert rel(y, ry) < 4e-3 and torch.allclose(r, rr, rtol=1e-5)


def test_swiglu():
    g = (torch.randn(1000, 1024, device="cuda") * 2).to(bf)
    u = torch.randn(1000, 1024, device="cuda").to(bf)
    assert rel(ew.swiglu_fwd(g, u), ew.ref_swiglu_fwd(g, u)) < 4e-3
    da = torch.randn(1000, 1024, device="cuda").to(bf)
    dg, du = ew.swiglu_bwd(da, g, u)
    rg, ru = ew.ref_swiglu_bwd(da, g, u)
    assert rel(dg, rg) < 4e-3 and rel(du, ru) < 4e-3
    # fused variant: in place over g/u, re-emits the activation bit-identically
    a_fwd = ew.swiglu_fwd(g, u)
    g2, u2, act = g.clone(), u.clone(), torch.empty_like(g)
    dg2, du2 = ew.swiglu_bwd(da, g2, u2, out_g=g2, out_u=u2, act_out=act)
    assert torch.equal(act, a_fwd)
    assert torch.equal(dg2, dg) and torch.equal(du2, du)


def test_rope_and_layout():
    from paper_2508_02932_b200.model import PRESETS, rope_tables
    B, s, H, hd = 3, 128, 4, 128
    cos, sin = rope_tables(PRESETS["llama-3.1-8b"], s, "cuda")
    x = torch.randn(B, s, H, hd, device="cuda").to(bf)
    out = ew.rope(x, cos, sin, s)
    assert rel(out.view(B, s, H, hd), ew.ref_rope(x, cos, sin)) < 4e-3
    back = ew.rope(out.view(B, s, H, hd), cos, sin, s, inverse=True)
    assert rel(back.view(B, s, H, hd), x) < 8e-3
    xt = torch.randn(B, H, s, hd, device="cuda").to(bf)   # SDPA-grad layout
    o = ew.rope(xt.transpose(1, 2), cos, sin, s, inverse=True)
    assert rel(o.view(B, s, H, hd), ew.ref_rope(xt.transpose(1, 2), cos, sin, inverse=True)) < 4e-3
    c = ew.rope(xt.transpose(1, 2), cos, sin, s, rotate=False)
    assert torch.equal(c.view(B, s, H, hd), xt.transpose(1, 2))
    inplace = x.clone().view(B * s, H * hd)
    ew.rope(inplace.view(B, s, H, hd), cos, sin, s, out=inplace)
    assert torch.equal(inplace, out)


@pytest.mark.parametrize("V", [1024, 128256, 151936, 1000])
def test_cross_entropy(V):
    logits = (torch.randn(64, V, device="cuda") * 3).to(bf)
    labels = torch.randint(0, V, (64,), device="cuda")
    weight = torch.rand(64, device="cuda")
    weight[5] = 0
    rg, rt = ew.ref_cross_entropy(logits, labels, weight)
    tok = torch.empty(64, device="cuda")
    g = logits.clone()
    ew.cross_entropy(g, labels, weight, tok)
    assert torch.allclose(tok, rt, rtol=1e-3, atol=1e-4)
    assert rel(g, rg) < 1e-2
    assert not torch.any(g[5])
