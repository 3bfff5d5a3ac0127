"""Packed LoRA linear at bench-like sizes through the torch-tensor ABI (ops.*),
checked against a torch fp32 reference of the same bf16 operands, plus
size-independent properties (linearity in alpha, packing invariance)."""

import numpy as np
import pytest
import torch

from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta

pytestmark = pytest.mark.gpu

bf = torch.bfloat16


def make(ranks, tokens, d, k, seed=0, kmajor=True):
    g = torch.Generator(device="cuda").manual_seed(seed)
    n = len(ranks)
    alphas = [float(r) * m for r, m in zip(ranks, [0.25, 1.0, 2.0, 4.0] * 8)]
    meta = build_meta(ranks, tokens, alphas).to("cuda")
    T = meta.total_tokens
    R64 = meta.rpad64
    x = torch.randn(T, d, device="cuda", generator=g).to(bf)
    w = (torch.randn(k, d, device="cuda", generator=g) * 0.02 if kmajor else
         torch.randn(d, k, device="cuda", generator=g) * 0.02).to(bf)
    a_sh = torch.zeros(n, d, R64, device="cuda", dtype=bf)
    bt_sh = torch.zeros(n, k, R64, device="cuda", dtype=bf)
    for i, r in enumerate(ranks):
        a_sh[i, :, :r] = ((torch.rand(d, r, device="cuda", generator=g) * 2 - 1) / d ** 0.5).to(bf)
        bt_sh[i, :, :r] = (torch.randn(k, r, device="cuda", generator=g) * 0.02).to(bf)
    dy = (torch.randn(T, k, device="cuda", generator=g) * 0.1).to(bf)
    return meta, x, w, a_sh, bt_sh, dy


def reference(meta, x, w, kmajor, a_sh, bt_sh, dy):
    W = w.float().t() if kmajor else w.float()
    y = x.float() @ W
    dx = dy.float() @ W.t()
    dA, dB, hs_all = [], [], []
    for i in range(meta.n_adapters):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        r = meta.ranks[i]
        al = meta.alphas[i]
        A = a_sh[i, :, :r].float()
        B = bt_sh[i, :, :r].float().t()
        xi, dyi = x[s:e].float(), dy[s:e].float()
        hs = (al * (xi @ A)).to(bf).float()          # the kernel stores Hs in bf16
        y[s:e] += hs @ B
        dh = (al * (dyi @ B.t())).to(bf).float()     # and dH in bf16
        dx[s:e] += dh @ A.t()
        dB.append(dyi.t() @ hs)                      # dB^T [k][r]
        dA.append(xi.t() @ dh)                       # dA [d][r]
        hs_all.append(hs)
    return y, dx, dA, dB


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


@pytest.mark.parametrize("kmajor", [True, False])
@pytest.mark.parametrize("d,k", [(4096, 4096), (4096, 1024), (1024, 3072)])
def test_packed_linear_vs_torch(kmajor, d, k):
    ranks = [8, 16, 32, 64]
    tokens = [1024, 512, 1024, 2048]
    meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, d, k, seed=d + k, kmajor=kmajor)
    y, hs = ops.linear_fwd(meta, x, w, kmajor, a_sh, bt_sh)
    R16 = meta.rpad16_total
    ga = torch.empty(d * R16, device="cuda")
    gb = torch.empty(k * R16, device="cuda")
    dx = ops.linear_bwd(meta, x, w, kmajor, a_sh, bt_sh, hs, dy, ga, gb)
    ry, rdx, rdA, rdB = reference(meta, x, w, kmajor, a_sh, bt_sh, dy)
    assert rel(y, ry) < 1e-2
    assert rel(dx, rdx) < 1e-2
    for i, r in enumerate(ranks):
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk_a = ga[d * int(meta.rpad_off[i]): d * int(meta.rpad_off[i + 1])].view(d, rp)
        blk_b = gb[k * int(meta.rpad_off[i]): k * int(meta.rpad_off[i + 1])].view(k, rp)
        assert rel(blk_a[:, :r], rdA[i]) < 5e-3, ("dA", i)
        assert rel(blk_b[:, :r], rdB[i]) < 5e-3, ("dB", i)
        assert not torch.any(blk_a[:, r:]) and not torch.any(blk_b[:, r:])   # padding stays zero


@pytest.mark.parametrize("kmajor", [True, False])
def test_unaligned_segments_pair_tiles(kmajor):
    """Segments that are not multiples of 128/256 rows (odd CTA-pair tiles, a 5-token
    segment, an empty one) through the CTA-pair GEMM (N >= 256) and the 1-CTA kernels."""
    ranks, tokens = [8, 64, 16, 32, 40], [300, 5, 0, 129, 700]
    d, k = 320, 512
    meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, d, k, seed=77, kmajor=kmajor)
    y, hs = ops.linear_fwd(meta, x, w, kmajor, a_sh, bt_sh)
    ga = torch.empty(d * meta.rpad16_total, device="cuda")
    gb = torch.empty(k * meta.rpad16_total, device="cuda")
    dx = ops.linear_bwd(meta, x, w, kmajor, a_sh, bt_sh, hs, dy, ga, gb)
    ry, rdx, rdA, rdB = reference(meta, x, w, kmajor, a_sh, bt_sh, dy)
    assert rel(y, ry) < 1e-2 and rel(dx, rdx) < 1e-2
    for i, r in enumerate(ranks):
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk_a = ga[d * int(meta.rpad_off[i]): d * int(meta.rpad_off[i + 1])].view(d, rp)
        blk_b = gb[k * int(meta.rpad_off[i]): k * int(meta.rpad_off[i + 1])].view(k, rp)
        if tokens[i] == 0:
            assert not torch.any(blk_a) and not torch.any(blk_b)
            continue
        assert rel(blk_a[:, :r], rdA[i]) < 5e-3, ("dA", i)
        assert rel(blk_b[:, :r], rdB[i]) < 5e-3, ("dB", i)


def _whole_tiles(meta):
    """plora_pack_t without a workspace: the LoRA kernels run whole tiles (no stream-K)."""
    s = meta.struct
    s.d_ws = None
    s.ws_bytes = 0
    return s


@pytest.mark.parametrize("stream_k", [False, True])
def test_packing_invariance(stream_k, monkeypatch):
    """Adapter i's outputs/grads in a pack equal running it alone.  With
    whole tiles bit for bit; with the stream-K LoRA kernels the split points of a tile
    depend on the rest of the pack, so the fp32 partial sums associate differently:
    equal to fp32 rounding (bf16 outputs within a last-bit flip)."""
    if not stream_k:
        monkeypatch.setattr(ops, "_pack", _whole_tiles)
    d, k = 1024, 2048
    ranks, tokens = [8, 64, 16], [256, 384, 128]
    meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, d, k, seed=5)
    y, hs = ops.linear_fwd(meta, x, w, True, a_sh, bt_sh)
    ga = torch.empty(d * meta.rpad16_total, device="cuda")
    gb = torch.empty(k * meta.rpad16_total, device="cuda")
    dx = ops.linear_bwd(meta, x, w, True, a_sh, bt_sh, hs, dy, ga, gb)
    for i in range(3):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        solo = build_meta([ranks[i]], [tokens[i]], [meta.alphas[i]], nb=meta.nb).to("cuda")
        ys, hss = ops.linear_fwd(solo, x[s:e].contiguous(), w, True, a_sh[i:i + 1].contiguous(),
                                 bt_sh[i:i + 1].contiguous())
        gas = torch.empty(d * solo.rpad16_total, device="cuda")
        gbs = torch.empty(k * solo.rpad16_total, device="cuda")
        dxs = ops.linear_bwd(solo, x[s:e].contiguous(), w, True, a_sh[i:i + 1].contiguous(),
                             bt_sh[i:i + 1].contiguous(), hss, dy[s:e].contiguous(), gas, gbs)
        off = int(meta.rpad_off[i])
        rp = solo.rpad16_total
        pairs = ((ys, y[s:e]), (dxs, dx[s:e]), (gas, ga[d * off: d * (off + rp)]), (gbs, gb[k * off: k * (off + rp)]))
        for got, want in pairs:
            if stream_k:
                assert rel(got, want) < 2e-3
            else:
                assert torch.equal(got, want)   # same tiles, same math: bit-identical


def test_deterministic_grads():
    meta, x, w, a_sh, bt_sh, dy = make([8, 16, 32, 64], [1024, 1024, 2048, 1024], 2048, 2048, seed=9)
    outs = []
    for _ in range(2):
        y, hs = ops.linear_fwd(meta, x, w, True, a_sh, bt_sh)
        ga = torch.empty(2048 * meta.rpad16_total, device="cuda")
        gb = torch.empty(2048 * meta.rpad16_total, device="cuda")
        dx = ops.linear_bwd(meta, x, w, True, a_sh, bt_sh, hs, dy, ga, gb)
        outs.append((y, dx, ga, gb))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_segred_lpt_schedule_matches_round_robin():
    """The LPT tile schedule (host row offsets present) and plain round-robin give
    bit-identical segment reductions: each output tile is still owned by one CTA."""
    ranks = [8, 64, 16, 32, 8, 64, 1, 48]
    tokens = [4096, 1024, 0, 2048, 333, 1024, 4096, 1500]
    for mdim in (4096, 1024, 14336):
        meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, mdim, 256, seed=3)
        q = (torch.randn(meta.total_tokens, meta.rpad64, device="cuda") * 0.1).to(bf)
        g_lpt = torch.full((mdim * meta.rpad16_total,), float("nan"), device="cuda")
        g_rr = torch.full_like(g_lpt, float("nan"))
        ops.segred(meta, x, q, g_lpt)
        saved = meta.struct.h_row_off
        meta.struct.h_row_off = None            # no host offsets -> round-robin schedule
        try:
            ops.segred(meta, x, q, g_rr)
        finally:
            meta.struct.h_row_off = saved
        torch.cuda.synchronize()
        assert not torch.isnan(g_lpt).any()
        assert torch.equal(g_lpt, g_rr)
        # and against the fp32 reference
        for i in range(meta.n_adapters):
            s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
            rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
            blk = g_lpt[mdim * int(meta.rpad_off[i]): mdim * int(meta.rpad_off[i + 1])].view(mdim, rp)
            ref = x[s:e].float().t() @ q[s:e, :rp].float()
            assert rel(blk, ref) < 1e-4 if e > s else torch.equal(blk, torch.zeros_like(blk))


@pytest.mark.parametrize("n_multi,big_rank", [(2, False), (3, False), (3, True)])
def test_multi_target_shrink_and_segred_match_single(n_multi, big_rank):
    """K2a / K5 over targets sharing their input (q/k/v, gate/up) in one launch equal the
    per-target launches bit for bit (same K order per output column); with a rank > 64
    (two 64-column rank blocks) the entry points fall back to per-target launches."""
    ranks = [8, 64, 16, 32, 8, 100 if big_rank else 64, 1, 48]
    tokens = [4096, 1024, 0, 2048, 333, 1024, 4096, 1500]
    d = 4096
    meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, d, 256, seed=5)
    T, R64 = meta.total_tokens, meta.rpad64
    g = torch.Generator(device="cuda").manual_seed(9)
    ls = [(torch.randn(meta.n_adapters, d, R64, device="cuda", generator=g) * 0.02).to(bf) for _ in range(n_multi)]
    outs = [torch.empty(T, R64, device="cuda", dtype=bf) for _ in range(n_multi)]
    ops.shrink_multi(meta, x, ls, outs)
    for l, o in zip(ls, outs):
        ref = torch.empty_like(o)
        ops.shrink(meta, x, l, ref)
        assert torch.equal(o, ref)
    qs = [(torch.randn(T, R64, device="cuda", generator=g) * 0.1).to(bf) for _ in range(n_multi)]
    gs = [torch.full((d * meta.rpad16_total,), float("nan"), device="cuda") for _ in range(n_multi)]
    ops.segred_multi(meta, x, qs, gs)
    for q, gm in zip(qs, gs):
        ref = torch.full_like(gm, float("nan"))
        ops.segred(meta, x, q, ref)
        assert torch.equal(gm, ref)


@pytest.mark.parametrize("kmajor,big_rank", [(True, False), (False, False), (True, True)])
def test_grouped_expand_and_dx_match_separate(kmajor, big_rank):
    """Grouped K1+K2b (N-segments, q/k/v-like widths incl. a narrow one) and grouped K6
    (K-segments: one fp32 accumulator) vs separate launches / the fp32 reference; a
    rank > 64 adds a second LoRA K-block per segment."""
    ranks = [8, 64, 16, 32, 8, 128 if big_rank else 64, 1, 48]
    tokens = [4096, 1024, 0, 2048, 333, 1024, 4096, 1500]
    d = 1024
    widths = [1024, 256, 512]
    meta = build_meta(ranks, tokens, [float(r) for r in ranks]).to("cuda")
    T, R64, n = meta.total_tokens, meta.rpad64, len(ranks)
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(T, d, device="cuda", generator=g).to(bf)
    ws = [((torch.randn(k, d, device="cuda", generator=g) if kmajor else torch.randn(d, k, device="cuda", generator=g))
           * 0.03).to(bf) for k in widths]
    bts = [(torch.randn(n, k, R64, device="cuda", generator=g) * 0.02).to(bf) for k in widths]
    ats = [(torch.randn(n, d, R64, device="cuda", generator=g) * 0.02).to(bf) for _ in widths]
    hss = [(torch.randn(T, R64, device="cuda", generator=g) * 0.5).to(bf) for _ in widths]
    for h in hss:                                    # rank padding columns are zero in real packs
        for i, r in enumerate(ranks):
            h[meta.row_offsets[i]:meta.row_offsets[i + 1], r:] = 0
    ys = ops.linear_expand_group(meta, x, ws, bts, hss, w_kmajor=kmajor)
    for w, bt, hs, y in zip(ws, bts, hss, ys):
        ref = ops.linear_expand(meta, x, w, kmajor, bt, hs)
        assert torch.equal(y, ref)
    dys = [(torch.randn(T, k, device="cuda", generator=g) * 0.1).to(bf) for k in widths]
    dx = ops.linear_dx_group(meta, dys, ws, ats, hss, d, w_kmajor=kmajor)
    want = torch.zeros(T, d, device="cuda")
    for w, at, dh, dy in zip(ws, ats, hss, dys):
        W = w.float().t() if kmajor else w.float()          # [d][k]
        want += dy.float() @ W.t()
        for i, r in enumerate(ranks):
            s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
            want[s:e] += dh[s:e, :r].float() @ at[i, :, :r].float().t()
    assert rel(dx, want) < 5e-3


@pytest.mark.parametrize("ffn", [1024, 1280, 1408])
def test_gate_up_swiglu_fused_matches_unfused(ffn):
    """gate/up K1+K2b with the SwiGLU forward in the epilogue == two grouped expands +
    swiglu_fwd, bit for bit (ffn not a multiple of 512 / 256 exercises partial tiles)."""
    from paper_2508_02932_b200 import elementwise as ew
    ranks = [8, 64, 16, 32, 1]
    tokens = [1024, 333, 2048, 0, 700]
    d = 512
    meta = build_meta(ranks, tokens, [2.0 * r for r in ranks]).to("cuda")
    T, R64, n = meta.total_tokens, meta.rpad64, len(ranks)
    g_ = torch.Generator(device="cuda").manual_seed(31)
    x = torch.randn(T, d, device="cuda", generator=g_).to(bf)
    wg, wu = [(torch.randn(ffn, d, device="cuda", generator=g_) * 0.05).to(bf) for _ in range(2)]
    btg, btu = [(torch.randn(n, ffn, R64, device="cuda", generator=g_) * 0.05).to(bf) for _ in range(2)]
    hsg, hsu = [(torch.randn(T, R64, device="cuda", generator=g_)).to(bf) for _ in range(2)]
    for h in (hsg, hsu):
        for i, r in enumerate(ranks):
            h[meta.row_offsets[i]:meta.row_offsets[i + 1], r:] = 0
    g, u, act = ops.linear_gate_up_swiglu(meta, x, wg, wu, btg, btu, hsg, hsu)
    rg, ru = ops.linear_expand_group(meta, x, [wg, wu], [btg, btu], [hsg, hsu])
    torch.cuda.synchronize()
    assert torch.equal(g, rg) and torch.equal(u, ru)
    assert torch.equal(act, ew.swiglu_fwd(rg, ru))


@pytest.mark.parametrize("widths", [[1024, 256, 512], [512, 128, 128]])
def test_grouped_expand_bias_epilogue(widths):
    """q/k/v biases added in the grouped GEMM epilogue (or by plora_add_row_bias when a
    narrow target forces separate launches) == the bf16 output + bf16 bias, bit for bit."""
    ranks, tokens = [8, 64, 16], [1024, 333, 700]
    d = 512
    meta = build_meta(ranks, tokens, [2.0 * r for r in ranks]).to("cuda")
    T, R64, n = meta.total_tokens, meta.rpad64, len(ranks)
    g = torch.Generator(device="cuda").manual_seed(41)
    x = torch.randn(T, d, device="cuda", generator=g).to(bf)
    ws = [(torch.randn(k, d, device="cuda", generator=g) * 0.05).to(bf) for k in widths]
    bts = [(torch.randn(n, k, R64, device="cuda", generator=g) * 0.05).to(bf) for k in widths]
    hss = [torch.randn(T, R64, device="cuda", generator=g).to(bf) for _ in widths]
    bs = [torch.randn(k, device="cuda", generator=g).to(bf) for k in widths]
    ys = ops.linear_expand_group(meta, x, ws, bts, hss, biases=bs)
    refs = ops.linear_expand_group(meta, x, ws, bts, hss)
    for y, r, b in zip(ys, refs, bs):
        assert torch.equal(y, r + b)


@pytest.mark.parametrize("d,k", [(4096, 14336), (14336, 4096)])
def test_full_c3_size_packed_linear(d, k):
    """BASELINE C3 at full size: the 16 bench adapters (ranks [8,16,32,64] x 4, batches
    1..4 x 1024 tokens, T = 32,768) through the gate/up (d=4096 -> k=14336) and down
    (14336 -> 4096) shapes, forward + backward, against the fp32 torch reference of the
    same bf16 operands (the bf16 tier: rel-Frobenius <= 1e-2 for Y / dX, 5e-3 for dA / dB)."""
    from paper_2508_02932_b200.model import bench_adapters
    specs, s = bench_adapters("llama-3.1-8b")
    ranks = [sp.rank for sp in specs]
    tokens = [sp.batch * s for sp in specs]
    meta, x, w, a_sh, bt_sh, dy = make(ranks, tokens, d, k, seed=d ^ k, kmajor=True)
    assert meta.total_tokens == 32768
    y, hs = ops.linear_fwd(meta, x, w, True, a_sh, bt_sh)
    ga = torch.empty(d * meta.rpad16_total, device="cuda")
    gb = torch.empty(k * meta.rpad16_total, device="cuda")
    dx = ops.linear_bwd(meta, x, w, True, a_sh, bt_sh, hs, dy, ga, gb)
    torch.backends.cuda.matmul.allow_tf32 = False
    ry, rdx, rdA, rdB = reference(meta, x, w, True, a_sh, bt_sh, dy)
    assert rel(y, ry) < 1e-2 and rel(dx, rdx) < 1e-2
    for i, r in enumerate(ranks):
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk_a = ga[d * int(meta.rpad_off[i]): d * int(meta.rpad_off[i + 1])].view(d, rp)
        blk_b = gb[k * int(meta.rpad_off[i]): k * int(meta.rpad_off[i + 1])].view(k, rp)
        assert rel(blk_a[:, :r], rdA[i]) < 5e-3, ("dA", i)
        assert rel(blk_b[:, :r], rdB[i]) < 5e-3, ("dB", i)
    # size-independent property: the LoRA part is linear in alpha -- doubling every alpha
    # doubles Y - X W exactly up to the bf16 rounding of Hs (checked at the same tolerance)
    meta2 = build_meta(ranks, tokens, [2 * a for a in meta.alphas]).to("cuda")
    y2, _ = ops.linear_fwd(meta2, x, w, True, a_sh, bt_sh)
    base = (x.float() @ w.float().t())
    assert rel(y2.float() - base, 2 * (ry - base)) < 2e-2


@pytest.mark.parametrize("d,widths,kmajor", [(4096, [4096, 1024, 1024], True), (4096, [14336, 14336], True),
                                             (4096, [4096, 1024, 1024], False)])
def test_grouped_ops_at_c3_widths(d, widths, kmajor):
    """The grouped pair launches at the C3 widths -- q/k/v (N-segments 4096/1024/1024 and
    their K-segmented input gradient) and gate/up (K-segments 14336 + 14336) -- take the
    256 x 512 (NB = 2) tiles: against separate launches and the fp32 reference."""
    ranks, tokens = [8, 16, 32, 64], [512, 256, 768, 512]
    meta = build_meta(ranks, tokens, [0.25 * 8, 16.0, 64.0, 256.0]).to("cuda")
    T, R64, n = meta.total_tokens, meta.rpad64, len(ranks)
    g = torch.Generator(device="cuda").manual_seed(77)
    x = torch.randn(T, d, device="cuda", generator=g).to(bf)
    ws = [((torch.randn(k, d, device="cuda", generator=g) if kmajor else torch.randn(d, k, device="cuda", generator=g))
           * 0.02).to(bf) for k in widths]
    bts = [(torch.randn(n, k, R64, device="cuda", generator=g) * 0.02).to(bf) for k in widths]
    ats = [(torch.randn(n, d, R64, device="cuda", generator=g) * 0.02).to(bf) for _ in widths]
    hss = [(torch.randn(T, R64, device="cuda", generator=g) * 0.5).to(bf) for _ in widths]
    for h in hss:
        for i, r in enumerate(ranks):
            h[meta.row_offsets[i]:meta.row_offsets[i + 1], r:] = 0
    if len(widths) == 3:
        ys = ops.linear_expand_group(meta, x, ws, bts, hss, w_kmajor=kmajor)
        for w, bt, hs, y in zip(ws, bts, hss, ys):
            W = w.float().t() if kmajor else w.float()
            want = x.float() @ W
            for i, r in enumerate(ranks):
                s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
                want[s:e] += hs[s:e, :r].float() @ bt[i, :, :r].float().t()
            assert rel(y, want) < 1e-2
            assert torch.equal(y, ops.linear_expand(meta, x, w, kmajor, bt, hs))
    dys = [(torch.randn(T, k, device="cuda", generator=g) * 0.1).to(bf) for k in widths]
    dx = ops.linear_dx_group(meta, dys, ws, ats, hss, d, w_kmajor=kmajor)
    want = torch.zeros(T, d, device="cuda")
    for w, at, dh, dy in zip(ws, ats, hss, dys):
        W = w.float().t() if kmajor else w.float()          # [d][k]
        want += dy.float() @ W.t()
        for i, r in enumerate(ranks):
            s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
            want[s:e] += dh[s:e, :r].float() @ at[i, :, :r].float().t()
    assert rel(dx, want) < 1e-2
