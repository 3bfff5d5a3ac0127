"""Stream-K partition of the LoRA kernels (K2a/K4 shrink, K3/K5 segment reductions):
every SM streams the same number of k-blocks and tiles cut by CTA boundaries are
summed by their last-arriving piece (gemm_sm100.cuh SkIter / sk_arrive / sk_gather).

Checked against the whole-tile schedule (pack without a workspace) and a torch fp32
reference of the same bf16 operands, on the shapes where the partition matters: one
adapter at T = 4096 (a rank's share of the 8-GPU planner split), tiny T (one tile cut
into up to 64 pieces), ranks > 64 (two rank blocks), empty segments."""

import pytest
import torch

from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta

pytestmark = pytest.mark.gpu

bf = torch.bfloat16

CASES = [
    ("split8-rank", [64], [4096], 4096),
    ("mixed", [8, 64, 16, 32, 8, 64, 1, 48], [4096, 1024, 0, 2048, 333, 1024, 4096, 1500], 4096),
    ("tiny", [16], [100], 4096),
    ("two-blocks", [100, 8], [700, 1300], 1024),
    ("ffn-width", [8, 16, 32, 64], [1024, 2048, 1024, 4096], 14336),
]


def _whole_tiles(meta):
    s = meta.struct
    s.d_ws = None
    s.ws_bytes = 0
    return s


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30))


def _operands(ranks, tokens, K, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    meta = build_meta(ranks, tokens, [0.5 + i for i in range(len(ranks))]).to("cuda")
    T, R64 = meta.total_tokens, meta.rpad64
    p = torch.randn(T, K, device="cuda", generator=g).to(bf)
    l_sh = torch.zeros(len(ranks), K, R64, device="cuda", dtype=bf)
    for i, r in enumerate(ranks):
        l_sh[i, :, :r] = (torch.randn(K, r, device="cuda", generator=g) / K ** 0.5).to(bf)
    q = (torch.randn(T, R64, device="cuda", generator=g) * 0.1).to(bf)
    return meta, p, l_sh, q


@pytest.mark.parametrize("name,ranks,tokens,K", CASES)
def test_shrink_stream_k(name, ranks, tokens, K, monkeypatch):
    meta, p, l_sh, _ = _operands(ranks, tokens, K, seed=1)
    T, R64 = meta.total_tokens, meta.rpad64
    sk = torch.empty(T, R64, device="cuda", dtype=bf)
    sk2 = torch.empty_like(sk)
    ops.shrink(meta, p, l_sh, sk)
    ops.shrink(meta, p, l_sh, sk2)
    with monkeypatch.context() as m:
        m.setattr(ops, "_pack", _whole_tiles)
        whole = torch.empty_like(sk)
        ops.shrink(meta, p, l_sh, whole)
    torch.cuda.synchronize()
    assert torch.equal(sk, sk2)                       # deterministic for a given pack
    assert rel(sk, whole) < 2e-3                      # same sums, other association (bf16 out)
    for i, r in enumerate(ranks):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        if e == s:
            continue
        ref = meta.alphas[i] * (p[s:e].float() @ l_sh[i, :, :r].float())
        assert rel(sk[s:e, :r], ref) < 1e-2, (name, i)
        assert not torch.any(sk[s:e, r:])            # zero-padded rank columns stay zero


@pytest.mark.parametrize("name,ranks,tokens,K", CASES)
def test_segred_stream_k(name, ranks, tokens, K, monkeypatch):
    meta, p, _, q = _operands(ranks, tokens, K, seed=2)
    Mdim = K
    g_sk = torch.full((Mdim * meta.rpad16_total,), float("nan"), device="cuda")
    g_sk2 = torch.full_like(g_sk, float("nan"))
    ops.segred(meta, p, q, g_sk)
    ops.segred(meta, p, q, g_sk2)
    with monkeypatch.context() as m:
        m.setattr(ops, "_pack", _whole_tiles)
        g_whole = torch.full_like(g_sk, float("nan"))
        ops.segred(meta, p, q, g_whole)
    torch.cuda.synchronize()
    assert not torch.isnan(g_sk).any()
    assert torch.equal(g_sk, g_sk2)
    assert rel(g_sk, g_whole) < 1e-5
    for i in range(meta.n_adapters):
        s, e = meta.row_offsets[i], meta.row_offsets[i + 1]
        rp = int(meta.rpad_off[i + 1] - meta.rpad_off[i])
        blk = g_sk[Mdim * int(meta.rpad_off[i]): Mdim * int(meta.rpad_off[i + 1])].view(Mdim, rp)
        if e == s:
            assert torch.equal(blk, torch.zeros_like(blk))
            continue
        ref = p[s:e].float().t() @ q[s:e, :rp].float()
        assert rel(blk, ref) < 1e-4, (name, i)


def test_workspace_left_zeroed():
    """The arrival counters are reset by the last piece of every split tile, so the
    workspace is reusable by the next launch on the stream without a memset."""
    meta, p, l_sh, q = _operands([16, 64], [100, 3000], 4096, seed=3)
    out = torch.empty(meta.total_tokens, meta.rpad64, device="cuda", dtype=bf)
    for _ in range(3):
        ops.shrink(meta, p, l_sh, out)
        ops.segred(meta, p, q, torch.empty(4096 * meta.rpad16_total, device="cuda"))
    torch.cuda.synchronize()
    ws = ops._workspace()
    assert not torch.any(ws[:1024])


def test_graph_replay_of_stream_k():
    """Captured in a CUDA graph (the workspace of the capture stream is created and
    zero-filled inside the capture), replays give the eager result."""
    meta, p, l_sh, q = _operands([64, 8], [2048, 2048], 4096, seed=4)
    eager = torch.empty(meta.total_tokens, meta.rpad64, device="cuda", dtype=bf)
    ops.shrink(meta, p, l_sh, eager)
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        ops.shrink(meta, p, l_sh, out)
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)
