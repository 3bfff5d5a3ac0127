import torch, torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel
B,H,KV,s,hd=32,32,8,1024,128
q=torch.randn(B,H,s,hd,device='cuda',dtype=torch.bfloat16,requires_grad=True)
k=torch.randn(B,KV,s,hd,device='cuda',dtype=torch.bfloat16,requires_grad=True)
v=torch.randn(B,KV,s,hd,device='cuda',dtype=torch.bfloat16,requires_grad=True)
do=torch.randn(B,H,s,hd,device='cuda',dtype=torch.bfloat16)
def t(fn,n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0,e1=torch.cuda.Event(True),torch.cuda.Event(True); e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)/n
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    f=t(lambda: F.scaled_dot_product_attention(q,k,v,is_causal=True,enable_gqa=True))
    fb=t(lambda: F.scaled_dot_product_attention(q,k,v,is_causal=True,enable_gqa=True).backward(do))
print(f"cudnn fwd {f:.3f} ms  fwd+bwd {fb:.3f} ms  bwd {fb-f:.3f} ms")
