"""Fused K3 + K4 (one pass over dY, ops.lora_dual / plora_lora_dual) against the separate
K4 shrink / K3 segment-reduction kernels and a torch fp32 reference of the reference's
Cases 2 and 1 (lorapack.py:225, :224): packs that take the fused path (several column
chunks, partial last m-tiles, an empty segment) and a pack too small for it (fallback)."""

import pytest
import torch

from paper_2508_02932_b200 import _lib, ops
from paper_2508_02932_b200.meta import build_meta

pytestmark = pytest.mark.gpu

bf = torch.bfloat16

C3_RANKS = [8, 16, 32, 64] * 4
C3_TOKENS = [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]
CASES = [
    ("c3-q", C3_RANKS, C3_TOKENS, 4096),
    ("c3-kv", C3_RANKS, C3_TOKENS, 1024),
    ("mixed", [8, 64, 16, 32, 8, 64, 1, 48], [4096, 1024, 0, 2048, 333, 1024, 4096, 1500], 2048),
    ("mixed-ffn", [8, 64, 16, 32, 8, 64, 1, 48], [4096, 1024, 0, 2048, 333, 1024, 4096, 1500], 14336),
    ("split8-rank", [64], [4096], 4096),   # a planner-split rank: 2-tile chunks x 8 column chunks
    ("tiny", [16], [100], 1024),          # one partial m-tile
]


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


def _operands(ranks, tokens, k, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    meta = build_meta(ranks, tokens, [0.25 * r for r in ranks]).to("cuda")
    T, R64 = meta.total_tokens, meta.rpad64
    dy = (torch.randn(T, k, device="cuda", generator=g)).to(bf)
    bt = torch.zeros(len(ranks), k, R64, device="cuda", dtype=bf)
    for i, r in enumerate(ranks):
        bt[i, :, :r] = (torch.randn(k, r, device="cuda", generator=g) * 0.02).to(bf)
    hs = torch.zeros(T, R64, device="cuda", dtype=bf)
    for i, r in enumerate(ranks):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        hs[s:e, :r] = torch.randn(e - s, r, device="cuda", generator=g).to(bf)
    return meta, dy, bt, hs


def _fused(meta, k):
    import ctypes
    s = meta.struct
    karr = (ctypes.c_int64 * 1)(k)
    return int(_lib.lib().plora_lora_dual_workspace_bytes(ctypes.byref(s), 1, karr, ops._h_rpad(meta))) > 0


@pytest.mark.parametrize("name,ranks,tokens,k", CASES)
def test_dual_matches_separate_and_fp32(name, ranks, tokens, k):
    meta, dy, bt, hs = _operands(ranks, tokens, k, seed=11)
    T, R64 = meta.total_tokens, meta.rpad64
    fused = _fused(meta, k)
    dh = torch.full((T, R64), float("nan"), device="cuda", dtype=bf)
    g = torch.full((k * meta.rpad16_total,), float("nan"), device="cuda")
    ops.lora_dual(meta, dy, bt, hs, dh, g)
    dh_sep = torch.empty_like(dh)
    g_sep = torch.full_like(g, float("nan"))
    ops.shrink(meta, dy, bt, dh_sep)
    ops.segred(meta, dy, hs, g_sep)
    torch.cuda.synchronize()
    assert not torch.isnan(dh).any() and not torch.isnan(g).any()
    if not fused:   # the plan chose the separate kernels: the same launches
        assert torch.equal(dh, dh_sep) and torch.equal(g, g_sep)
        return
    assert rel(g, g_sep) < 1e-5                       # same sums, other association (fp32)
    assert rel(dh, dh_sep) < 2e-3                     # bf16 outputs within a last-bit flip
    for i, r in enumerate(ranks):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk = g[k * int(meta.rpad_off[i]): k * int(meta.rpad_off[i + 1])].view(k, rp)
        if e == s:
            assert not torch.any(blk)
            continue
        ref_b = dy[s:e].float().t() @ hs[s:e, :rp].float()           # Case 1: dB^T = Hs^T dY
        ref_h = meta.alphas[i] * (dy[s:e].float() @ bt[i, :, :r].float())   # Case 2: dH = alpha dY B^T
        assert rel(blk, ref_b) < 1e-4, (name, i)
        assert rel(dh[s:e, :r], ref_h) < 5e-3, (name, i)
        assert not torch.any(dh[s:e, r:]), (name, i)    # zero past the rank (B zero-padded)


def test_dual_deterministic_and_graph_capturable():
    meta, dy, bt, hs = _operands(C3_RANKS, C3_TOKENS, 4096, seed=12)
    T, R64 = meta.total_tokens, meta.rpad64
    outs = []
    for _ in range(2):
        dh = torch.empty((T, R64), device="cuda", dtype=bf)
        g = torch.empty((4096 * meta.rpad16_total,), device="cuda")
        ops.lora_dual(meta, dy, bt, hs, dh, g)
        outs.append((dh, g))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    dh = torch.empty((T, R64), device="cuda", dtype=bf)
    g = torch.empty((4096 * meta.rpad16_total,), device="cuda")
    ops.lora_dual(meta, dy, bt, hs, dh, g)   # workspace sized outside the capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ops.lora_dual(meta, dy, bt, hs, dh, g)
    dh.zero_()
    g.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(dh, outs[0][0]) and torch.equal(g, outs[0][1])


def test_trainer_fused_dual_matches_separate():
    """One C1-shaped training step with and without the fused dY pass: same losses, LoRA
    grads equal to fp32 association (tiny packs take the separate path; a wider tiny
    model exercises the fused one)."""
    from paper_2508_02932_b200.model import ModelConfig, PackedLoraTrainer, bench_adapters

    cfg = ModelConfig(name="tiny-wide", d=512, n_layers=2, ffn=1536, n_heads=4, n_kv=4, vocab=1024,
                      tied=False, qkv_bias=False)
    specs, s = bench_adapters("tiny")
    specs = [type(sp)(rank=sp.rank, alpha=sp.alpha, batch=sp.batch * 16, lr=sp.lr) for sp in specs]
    res = []
    for fuse in (True, False):
        torch.manual_seed(0)
        tr = PackedLoraTrainer(cfg, specs, s, device="cuda", a_scale=0.05, b_std=0.05, fuse_dual=fuse)
        tokens = tr.synthetic_tokens().cuda()
        losses = tr.forward_backward(tokens).float().clone()
        res.append((losses, tr.bank.G.clone()))
    assert rel(res[0][0], res[1][0]) < 1e-6
    # dA inherits the bf16 rounding of dH (a last-bit flip where the fp32 sums associate
    # differently): ~1e-3 relative; dB itself agrees to fp32 association
    assert rel(res[0][1], res[1][1]) < 5e-3


PACKS = {"c3": (C3_RANKS, C3_TOKENS), "split8-1": ([64], [4096]), "split8-3": ([8, 32, 32], [1024, 2048, 1024])}


@pytest.mark.parametrize("pack", list(PACKS))
@pytest.mark.parametrize("ks", [(4096, 1024, 1024), (14336, 14336)])
def test_dual_multi_target_one_launch(ks, pack):
    """The q/k/v (or gate/up) targets of a layer in ONE fused launch equal the separate
    K4 / K3 kernels per target (fp32 association) -- on C3 and on planner-split rank packs,
    whose jointly planned launches mix targets of different unit sizes."""
    import ctypes
    ranks, tokens = PACKS[pack]
    meta = None
    dys, bts, hss = [], [], []
    for j, k in enumerate(ks):
        m, dy, bt, hs = _operands(ranks, tokens, k, seed=20 + j)
        meta = meta or m
        dys.append(dy), bts.append(bt), hss.append(hs)
    T, R64 = meta.total_tokens, meta.rpad64
    karr = (ctypes.c_int64 * len(ks))(*ks)
    assert int(_lib.lib().plora_lora_dual_workspace_bytes(ctypes.byref(meta.struct), len(ks), karr,
                                                          ops._h_rpad(meta))) > 0
    dhs = [torch.full((T, R64), float("nan"), device="cuda", dtype=bf) for _ in ks]
    gs = [torch.full((k * meta.rpad16_total,), float("nan"), device="cuda") for k in ks]
    ops.lora_dual(meta, dys, bts, hss, dhs, gs)
    for dy, bt, hs, dh, g, k in zip(dys, bts, hss, dhs, gs, ks):
        dh_sep = torch.empty_like(dh)
        g_sep = torch.empty_like(g)
        ops.shrink(meta, dy, bt, dh_sep)
        ops.segred(meta, dy, hs, g_sep)
        torch.cuda.synchronize()
        assert not torch.isnan(dh).any() and not torch.isnan(g).any()
        assert rel(g, g_sep) < 1e-5, k
        assert rel(dh, dh_sep) < 2e-3, k


def test_trainer_overlap_k5_identical_eager_and_graph():
    """dA reductions on the side stream (overlap_k5): the same kernels on the same data,
    so losses and every gradient are bit-identical to stream order, eager and replayed
    from a CUDA graph (the side stream joins before the optimizer)."""
    from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters

    specs, s = bench_adapters("tiny")
    res = []
    for overlap in (False, True):
        tr = PackedLoraTrainer(PRESETS["tiny"], specs, s, device="cuda", a_scale=0.05, b_std=0.05,
                               overlap_k5=overlap)
        tokens = tr.synthetic_tokens().cuda()
        losses = tr.forward_backward(tokens).float().clone()
        res.append((losses, tr.bank.G.clone()))
        if overlap:
            g = tr.graphed(tokens, warmup=1)
            g.graph.replay()
            torch.cuda.synchronize()
            tr2 = PackedLoraTrainer(PRESETS["tiny"], specs, s, device="cuda", a_scale=0.05, b_std=0.05)
            tr2.step(tokens)          # same warm-up step as the graphed trainer's
            l2 = tr2.forward_backward(tokens).float().clone()
            assert torch.equal(g.losses.float(), l2)
            assert torch.equal(tr.bank.G, tr2.bank.G)
    assert torch.equal(res[0][0], res[1][0])
    assert torch.equal(res[0][1], res[1][1])
