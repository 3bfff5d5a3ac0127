"""K7 fused per-adapter AdamW vs torch.optim.AdamW (fp32), one optimizer per adapter
with that adapter's learning rate (parity unpinned by the reference, which has no
optimizer; oracle = torch)."""

import pytest
import torch

from paper_2508_02932_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("device_steps", [False, True])
def test_adamw_matches_torch(device_steps):
    """device_steps: step = 0, each adapter's step count read from hp[i].z on the device
    (the graph-replayable form; the adapters start at different counts)."""
    torch.manual_seed(0)
    rows, rpads, sh_ld = [37, 64, 5], [16, 32, 64], 64
    lrs, wds = [1e-3, 5e-4, 2e-3], [0.0, 0.01, 0.1]
    n = len(rows)
    sizes = [r * p for r, p in zip(rows, rpads)]
    offs = [0]
    for s in sizes:
        offs.append(offs[-1] + s)
    P = torch.randn(offs[-1], device="cuda")
    M = torch.zeros_like(P)
    V = torch.zeros_like(P)
    shadow = torch.zeros(n, max(rows), sh_ld, device="cuda", dtype=torch.bfloat16)
    chunks = []
    for i in range(n):   # split adapter i's block into 2 row-chunks to exercise the table
        half = rows[i] // 2 or rows[i]
        for r0, r1 in ((0, half), (half, rows[i])):
            if r1 <= r0:
                continue
            chunks.append([offs[i] + r0 * rpads[i], i * max(rows) * sh_ld + r0 * sh_ld,
                           (r1 - r0) | (rpads[i] << 32), i | (sh_ld << 32)])
    chunks = torch.tensor(chunks, dtype=torch.int64, device="cuda")
    hp = torch.tensor([[lr, wd, 0.0, 0.0] for lr, wd in zip(lrs, wds)], device="cuda")
    ref = [torch.nn.Parameter(P[offs[i]:offs[i + 1]].clone()) for i in range(n)]
    opts = [torch.optim.AdamW([ref[i]], lr=lrs[i], weight_decay=wds[i], foreach=False) for i in range(n)]
    if device_steps:   # adapter i has already taken 2 * i steps (zero gradients: state unchanged but counted)
        for i in range(n):
            for _ in range(2 * i):
                ref[i].grad = torch.zeros_like(ref[i])
                opts[i].step()
            M[offs[i]:offs[i + 1]] = opts[i].state[ref[i]]["exp_avg"] if 2 * i else 0.0
            V[offs[i]:offs[i + 1]] = opts[i].state[ref[i]]["exp_avg_sq"] if 2 * i else 0.0
            P[offs[i]:offs[i + 1]] = ref[i].detach()
            hp[i, 2] = float(2 * i)
    for step in range(1, 6):
        G = torch.randn_like(P)
        if device_steps:
            hp[:, 2] += 1.0
            ops.adamw(chunks, P, G, M, V, shadow, hp, 0)
        else:
            ops.adamw(chunks, P, G, M, V, shadow, hp, step)
        for i in range(n):
            ref[i].grad = G[offs[i]:offs[i + 1]].clone()
            opts[i].step()
    for i in range(n):
        got = P[offs[i]:offs[i + 1]]
        assert torch.allclose(got, ref[i].detach(), rtol=1e-5, atol=1e-6), i
        sh = shadow[i, :rows[i], :rpads[i]].float().reshape(-1)
        assert torch.equal(sh, got.to(torch.bfloat16).float())
        assert not torch.any(shadow[i, :, rpads[i]:])
