import sys, torch
sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops
from paper_2508_02932_b200.meta import build_meta
bf = torch.bfloat16
def whole(meta):
    s = meta.struct; s.d_ws = None; s.ws_bytes = 0; return s
for (ranks, tokens, K) in [([64], [4096], 4096), ([16], [100], 4096), ([64], [4096], 256), ([64], [1024], 4096)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    meta = build_meta(ranks, tokens, [1.0]*len(ranks)).to("cuda")
    T = meta.total_tokens
    p = torch.randn(T, K, device="cuda", generator=g).to(bf)
    l = (torch.randn(len(ranks), K, meta.rpad64, device="cuda", generator=g) / K**0.5).to(bf)
    ref = (p.float() @ l[0].float())
    sk = torch.empty(T, meta.rpad64, device="cuda", dtype=bf)
    ops.shrink(meta, p, l, sk)
    orig = ops._pack
    ops._pack = whole
    wh = torch.empty_like(sk); ops.shrink(meta, p, l, wh)
    ops._pack = orig
    torch.cuda.synchronize()
    err_t = [(float((sk[i:i+128].float()-ref[i:i+128]).norm()/ref[i:i+128].norm())) for i in range(0, T, 128)]
    err_w = [(float((wh[i:i+128].float()-ref[i:i+128]).norm()/ref[i:i+128].norm())) for i in range(0, T, 128)]
    print(ranks, tokens, K, "sk per-tile err", [round(e, 3) for e in err_t][:40])
    print("   whole per-tile err", [round(e, 3) for e in err_w][:10])
    # ratio sk/ref per tile: is it a multiple (missing/duplicated pieces)?
    for i in range(0, min(T, 4 * 128), 128):
        a = sk[i:i+128].float().flatten(); b = ref[i:i+128].flatten()
        print("   tile", i // 128, "scale sk/ref", float((a * b).sum() / (b * b).sum()))
    ws = ops._workspace(); print("   counters nonzero:", int(torch.count_nonzero(ws[:1024])))
