"""FmhaBackward (CuTe-DSL Blackwell FMHA backward, attn_bwd.py) vs cuDNN SDPA's own backward
on trainer shapes, from cuDNN's forward output + log-sum-exp; prints max errors and times."""
import sys
import time

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, ".")
from paper_2508_02932_b200.attn_bwd import FmhaBackward  # noqa: E402


def ev_time(fn, n=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (b, s, H, KV, hd) in [(32, 1024, 32, 8, 128), (3, 128, 4, 4, 64), (4, 1024, 5, 1, 128), (8, 1024, 16, 2, 128)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    T = b * s
    q = torch.randn(T, H * hd, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(T, KV * hd, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(T, KV * hd, device="cuda", generator=g).to(torch.bfloat16)
    do = torch.randn(T, H * hd, device="cuda", generator=g).to(torch.bfloat16)
    qg = q.view(b, s, H, hd).transpose(1, 2)
    kg = k.view(b, s, KV, hd).transpose(1, 2)
    vg = v.view(b, s, KV, hd).transpose(1, 2)
    try:
        res = torch.ops.aten._scaled_dot_product_cudnn_attention(qg, kg, vg, None, True, 0.0, True, False)
        out, lse = res[0], res[1]
        gqa_native = True
    except Exception as e:   # noqa: BLE001
        print("aten cudnn op with GQA failed:", str(e)[:200])
        gqa_native = False
        continue
    print(f"shape b={b} s={s} H={H} KV={KV} hd={hd}: out {tuple(out.shape)} strides {out.stride()} "
          f"lse {tuple(lse.shape)} {lse.dtype} strides {lse.stride()}")
    o_tm = out.transpose(1, 2).reshape(T, H * hd)
    # reference: cuDNN autograd
    qr, kr, vr = (t.detach().clone().requires_grad_() for t in (qg, kg, vg))
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        outr = F.scaled_dot_product_attention(qr, kr, vr, is_causal=True, enable_gqa=(KV != H))
        outr.backward(do.view(b, s, H, hd).transpose(1, 2))
    print("  fwd out vs F.sdpa:", (outr.detach() - out).abs().max().item())
    fb = FmhaBackward(H, KV, hd)
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    t0 = time.time()
    fb(q, k, v, o_tm.contiguous(), do, lse.contiguous(), dq, dk, dv, b, s)
    torch.cuda.synchronize()
    print(f"  first call (compile) {time.time() - t0:.1f} s")
    for name, got, ref in (("dq", dq, qr.grad), ("dk", dk, kr.grad), ("dv", dv, vr.grad)):
        ref_tm = ref.transpose(1, 2).reshape(T, -1).float()
        err = (got.float() - ref_tm).abs().max().item()
        rel = ((got.float() - ref_tm).norm() / ref_tm.norm()).item()
        print(f"  {name}: max abs err {err:.3e}  rel fro {rel:.3e}  ref max {ref_tm.abs().max().item():.3e}")
    oc, lc = o_tm.contiguous(), lse.contiguous()
    t_cute = ev_time(lambda: fb(q, k, v, oc, do, lc, dq, dk, dv, b, s))
    dog = do.view(b, s, H, hd).transpose(1, 2)
    qr2, kr2, vr2 = (t.detach().clone().requires_grad_() for t in (qg, kg, vg))
    with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
        t_f = ev_time(lambda: F.scaled_dot_product_attention(qr2, kr2, vr2, is_causal=True, enable_gqa=(KV != H)))
        t_fb = ev_time(lambda: F.scaled_dot_product_attention(qr2, kr2, vr2, is_causal=True,
                                                              enable_gqa=(KV != H)).backward(dog))
    print(f"  bwd time: cute {t_cute:.3f} ms, cudnn {t_fb - t_f:.3f} ms (fwd {t_f:.3f} ms)")
