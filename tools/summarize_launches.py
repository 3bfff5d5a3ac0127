"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel shares."""
import csv
import json
import re
import sys
from collections import defaultdict


def classify(name: str) -> str:
    m = re.search(r"plora_gemm_pair_kernel<\(bool\)(\d), \(int\)(\d)>|plora_gemm_pair_kernel<(\w+), (\d)>", name)
    if "plora_gemm_pair_kernel" in name:
        return "gemm_pair (K1/K2b fwd, K6 dX, lm_head)"
    if "plora_swiglu_segred" in name:
        return "SwiGLU bwd + dA_down (fused)"
    if "plora_dual" in name:
        return "dual K4+K3 (one dY pass + fix-up)"
    if "plora_segred_lpt_kernel" in name:
        return "segred (K3/K5)"
    if "plora_gemm_kernel" in name:
        if ", 1," in name or "(int)1," in name:
            return "shrink (K2a/K4)"
        if ", 2," in name or "(int)2," in name:
            return "segred (K3/K5)"
        return "gemm_1cta (N<256)"
    for key in ("adamw", "add_rmsnorm", "rmsnorm_fwd", "rmsnorm_bwd", "swiglu_fwd", "swiglu_bwd", "rope", "ce_kernel",
                "ce_stats", "ce_apply"):
        if key in name:
            return key
    if "sdpa" in name or "fmha" in name or "cudnn" in name or "attention" in name:
        return "attention (cuDNN SDPA)"
    return "torch/other"


def main(path: str, out: str | None = None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        k = classify(d["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ns
        total += ns
    summary = {k: {"launches": c, "ms": round(t / 1e6, 3), "share": round(t / total, 4)}
               for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    summary["_total_ms"] = round(total / 1e6, 3)
    txt = json.dumps(summary, indent=1)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
