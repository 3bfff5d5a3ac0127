"""LoRA-kernel micro-benchmark: K2a/K4 shrink and K3/K5 segment reductions at the C3
pack (16 adapters, T = 32768) and at one rank's share of the 8-GPU planner split (one
rank-64 adapter, T = 4096), with the stream-K partition (pack workspace) and with whole
tiles.  CUDA events, warmed, L2 flushed between reps; GB/s = algorithmic bytes / time.

  python tools/bench_lora.py [--only NAME]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_02932_b200 import ops  # noqa: E402
from paper_2508_02932_b200.meta import build_meta  # noqa: E402

bf = torch.bfloat16
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
PEAK = 6549.4


def whole(meta):
    s = meta.struct
    s.d_ws = None
    s.ws_bytes = 0
    return s


def timeit(fn, reps=20, warm=3):
    """Median device time of fn: all reps are enqueued behind a 50 ms sleep kernel, so the
    events time the kernel back to back (no host launch latency inside the bracket)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(50e-3 * 1.9e9))
    evs = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    ts = sorted(s.elapsed_time(e) for s, e in evs)
    return ts[len(ts) // 2]


PACKS = {
    "c3": ([8, 16, 32, 64] * 4, [x * 1024 for x in [1, 1, 2, 4, 2, 1, 4, 1, 1, 2, 1, 4, 4, 2, 1, 1]]),
    "split8": ([64], [4096]),
}


def main():
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    out = {}
    for pname, (ranks, tokens) in PACKS.items():
        meta = build_meta(ranks, tokens, [1.0] * len(ranks)).to("cuda")
        T, R64 = meta.total_tokens, meta.rpad64
        tr, R = sum(t * r for t, r in zip(tokens, ranks)), sum(ranks)
        for K in (1024, 4096, 14336):
            name = f"{pname}_K{K}"
            if only and only not in name:
                continue
            p = torch.randn(T, K, device="cuda").to(bf)
            l_sh = (torch.randn(len(ranks), K, R64, device="cuda") * 0.01).to(bf)
            q = (torch.randn(T, R64, device="cuda") * 0.1).to(bf)
            hs = torch.empty(T, R64, device="cuda", dtype=bf)
            g = torch.empty(K * meta.rpad16_total, device="cuda")
            sh_bytes = 2.0 * T * K + 2.0 * K * R + 2.0 * tr
            sg_bytes = 2.0 * T * K + 2.0 * tr + 4.0 * K * R
            row = {}
            for mode in ("stream_k", "whole"):
                orig = ops._pack
                if mode == "whole":
                    ops._pack = whole
                try:
                    t_sh = timeit(lambda: ops.shrink(meta, p, l_sh, hs))
                    t_sg = timeit(lambda: ops.segred(meta, p, q, g))
                finally:
                    ops._pack = orig
                row[mode] = {"shrink_us": round(t_sh * 1e3, 1), "shrink_gbs": round(sh_bytes / t_sh / 1e6),
                             "segred_us": round(t_sg * 1e3, 1), "segred_gbs": round(sg_bytes / t_sg / 1e6)}
            dh = torch.empty(T, R64, device="cuda", dtype=bf)
            t_du = timeit(lambda: ops.lora_dual(meta, p, l_sh, q, dh, g))
            row["dual_us"] = round(t_du * 1e3, 1)
            row["dual_gbs_equiv"] = round((sh_bytes + sg_bytes) / t_du / 1e6)   # the two separate passes' bytes
            out[name] = row
            print(name, json.dumps(row), flush=True)
    print(json.dumps({"lora_kernels": out, "peak_gbs": PEAK}))


if __name__ == "__main__":
    main()
