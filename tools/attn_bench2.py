"""cuDNN SDPA fwd+bwd on the C3 attention shape under different input layouts / GQA handling."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, KV, s, hd = 32, 32, 8, 1024, 128


def run(name, q, k, v, gqa):
    do = torch.randn(B, H, s, hd, device="cuda", dtype=torch.bfloat16)
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        for _ in range(3):
            F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=gqa).backward(do)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=gqa).backward(do)
        e1.record()
        torch.cuda.synchronize()
    print(f"{name}: fwd+bwd {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)


def mk(shape_bshd, contiguous_bhsd):
    b, s_, h, d = shape_bshd
    if contiguous_bhsd:
        return torch.randn(b, h, s_, d, device="cuda", dtype=torch.bfloat16).requires_grad_()
    return torch.randn(b, s_, h, d, device="cuda", dtype=torch.bfloat16).transpose(1, 2).detach().requires_grad_()


run("BSHD views, GQA", mk((B, s, H, hd), False), mk((B, s, KV, hd), False), mk((B, s, KV, hd), False), True)
run("BHSD contiguous, GQA", mk((B, s, H, hd), True), mk((B, s, KV, hd), True), mk((B, s, KV, hd), True), True)
run("BSHD views, no GQA (H kv heads)", mk((B, s, H, hd), False), mk((B, s, H, hd), False), mk((B, s, H, hd), False),
    False)
