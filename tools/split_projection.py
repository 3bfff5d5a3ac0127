"""Planner-split scaling on ONE GPU: every rank's packed job of the N-GPU split
(sweep/jobsplit.py, the split bench.py --gpus N runs) trained here one after the other,
device-timed like bench.py.  Ranks of a real N-GPU run are independent processes on
their own GPUs with no data-path collective, so the N-GPU step time is the slowest
rank's: projected tokens/s = total tokens / max_r(step time of rank r).  A projection,
not a bench value (one GPU, ranks timed sequentially, no cross-rank interference).

  python tools/split_projection.py [--config llama-3.1-8b] [--gpus 2,4,8] [--steps 5] [--warmup 2]
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")

import torch  # noqa: E402

from paper_2508_02932_b200.model import PRESETS, PackedLoraTrainer, bench_adapters  # noqa: E402
from paper_2508_02932_b200.sweep.engine import _base  # noqa: E402
from paper_2508_02932_b200.sweep.jobsplit import split_adapters  # noqa: E402


TRAINER_KW = {}


def time_job(cfg_name, idx, steps, warmup, kernels=False, graph=False):
    cfg = PRESETS[cfg_name]
    specs, s = bench_adapters(cfg_name)
    sub = [specs[i] for i in idx]
    tr = PackedLoraTrainer(cfg, sub, s, device="cuda", base=_base(cfg_name, "cuda:0"),
                           adapter_seeds=[100 + i for i in idx], **TRAINER_KW)
    tok = tr.synthetic_tokens(seeds=[1000 + i for i in idx]).cuda()
    for _ in range(warmup):
        tr.step(tok)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    gs = tr.graphed(tok, warmup=1) if graph else None
    run = gs.step if graph else (lambda: tr.step(tok))
    torch.cuda.synchronize()
    e0.record()
    h0 = time.perf_counter()
    for _ in range(steps):
        run()
    host_ms = (time.perf_counter() - h0) * 1000 / steps   # host enqueue time (CPU-bound if ~ device time)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    T = tr.T
    del run, gs   # the timer graph below needs the memory of the step graph's pool
    torch.cuda.empty_cache()
    if kernels:   # per kernel class ms / step: the step captured with event-record nodes around every
        # libplora launch (device times, no host gaps; as bench.py's kernel stats), one replay
        from paper_2508_02932_b200 import ops
        timer = ops.KernelTimer(external=True)
        ops.set_timer(timer)
        try:
            tg = tr.graphed(tok, warmup=0)
        finally:
            ops.set_timer(None)
        tg.step()
        torch.cuda.synchronize()
        tg.step()
        summ = timer.summary()
        del tg
        print(json.dumps({"job": list(idx), "T": T, "ms_per_step": round(ms, 2), "host_ms_per_step": round(host_ms, 2),
                          "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 2)}
                                      for k, v in summ.items()}}), flush=True)
    del tr
    torch.cuda.empty_cache()
    return T, ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="llama-3.1-8b")
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--kernels", action="store_true", help="print each job's per-kernel-class times")
    ap.add_argument("--overlap-k5", action="store_true", help="trainer option overlap_k5 (A/B)")
    ap.add_argument("--no-overlap-k5", action="store_true", help="trainer option overlap_k5=False (A/B)")
    ap.add_argument("--graph", action="store_true", help="time the step replayed from a CUDA graph")
    ap.add_argument("--whole-lora", action="store_true",
                    help="A/B: LoRA kernels without the pack workspace (whole tiles, no stream-K)")
    args = ap.parse_args()
    if args.overlap_k5:
        TRAINER_KW["overlap_k5"] = True
    if args.no_overlap_k5:
        TRAINER_KW["overlap_k5"] = False
    if args.whole_lora:
        from paper_2508_02932_b200 import ops

        def whole(meta):
            s = meta.struct
            s.d_ws = None
            s.ws_bytes = 0
            return s
        ops._pack = whole
    torch.cuda.set_device(0)
    cache = {}
    out = {"config": args.config, "step_mode": "cuda_graph" if args.graph else "eager", "projection": []}
    one = None
    for n in [int(x) for x in args.gpus.split(",")]:
        sp = split_adapters(args.config, n)
        ranks = []
        for r, idx in enumerate(sp.adapters):
            key = tuple(idx)
            if key not in cache:
                cache[key] = time_job(args.config, list(idx), args.steps, args.warmup, args.kernels, args.graph)
            T, ms = cache[key]
            ranks.append({"rank": r, "adapters": list(idx), "tokens": T, "ms_per_step": round(ms, 2),
                          "tokens_per_s": round(T / ms * 1000, 1)})
        total = sum(x["tokens"] for x in ranks)
        step = max(x["ms_per_step"] for x in ranks)
        v = total / step * 1000
        if n == 1:
            one = v
        row = {"gpus": n, "split": sp.describe(), "projected_tokens_per_s": round(v, 1),
               "slowest_rank_ms": step, "efficiency_vs_1gpu": round(v / (n * one), 4) if one else None,
               "ranks": ranks}
        out["projection"].append(row)
        print(json.dumps({k: row[k] for k in ("gpus", "split", "projected_tokens_per_s", "slowest_rank_ms",
                                                "efficiency_vs_1gpu")}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
