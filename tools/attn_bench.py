"""SDPA backends on the C3 attention shape (B=32 sequences, 32 q heads / 8 kv heads,
s=1024, hd=128, causal, bf16): forward + backward time per backend."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, H, KV, s, hd = 32, 32, 8, 1024, 128
q = torch.randn(B, s, H, hd, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_()
k = torch.randn(B, s, KV, hd, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_()
v = torch.randn(B, s, KV, hd, device="cuda", dtype=torch.bfloat16).transpose(1, 2).requires_grad_()
do = torch.randn(B, H, s, hd, device="cuda", dtype=torch.bfloat16)
for be in [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION]:
    try:
        with sdpa_kernel(be):
            for _ in range(3):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
                o.backward(do)
            torch.cuda.synchronize()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record()
            for _ in range(5):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            e1.record()
            for _ in range(5):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
                o.backward(do)
            e2.record()
            torch.cuda.synchronize()
            f = e0.elapsed_time(e1) / 5
            fb = e1.elapsed_time(e2) / 5
            print(f"{be}: fwd {f:.3f} ms, fwd+bwd {fb:.3f} ms, o strides {o.stride()}")
    except Exception as ex:  # noqa: BLE001
        print(f"{be}: unavailable ({str(ex)[:120]})")
