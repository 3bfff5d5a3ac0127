"""Per-shape DRAM traffic of one timed bench step: an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum, timed
region only: PLORA_PROFILE_RANGE=1 + --profile-from-start off) matched launch by launch
with bench.py's own records of the same step (PLORA_RECORDS_OUT: kind, shape, algorithmic
flops / bytes per launch, in issue order).  Writes per-shape DRAM bytes vs algorithmic
bytes and the dominant GEMM launch's traffic (profiles/gemm_traffic.json, read by
bench.py for roofline.traffic).

  python tools/dram_by_shape.py launches.csv records.json out.json [gemm_traffic.json]
"""
import csv
import json
import sys
from collections import OrderedDict

TIMED = ("plora_gemm_pair_kernel", "plora_gemm_kernel", "plora_segred_lpt_kernel", "adamw_kernel", "plora_dual",
         "plora_swiglu_segred")
# launches per record: the fused K3+K4 pass is the dual kernel + its fix-up (or, for packs
# too small for it, the separate shrink + segment reduction)
PER_RECORD = {"dual": 2}
UNITS = {"ns": 1.0, "nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d.get("Metric Unit", ""), 1.0)
        per.setdefault(key, {})[d["Metric Name"]] = v
    return [(name, m) for (_, name), m in per.items()]


def main(lpath, rpath, out, traffic_out=None):
    ls = [(n, m) for n, m in launches(lpath) if any(k in n for k in TIMED)]
    recs = json.load(open(rpath))
    def per(r):   # the fused pass: dual + fix-up; its separate fallback: shrink + segred per target
        if r["kind"] == "dual" and str(r["detail"]).endswith("sep"):
            return 2 * (str(r["detail"]).count("+") + 1)
        return PER_RECORD.get(r["kind"], 1)
    need = sum(per(r) for r in recs)
    if len(ls) != need:
        raise SystemExit(f"{len(ls)} timed-kernel launches in the ncu list but {need} for the bench records")
    pairs, i = [], 0
    for r in recs:
        k = per(r)
        grp = ls[i:i + k]
        i += k
        m = {key: sum(g[1].get(key, 0.0) for g in grp) for key in grp[0][1]}
        pairs.append(((grp[0][0], m), r))
    agg = OrderedDict()
    for (name, m), r in pairs:
        key = f"{r['kind']}[{r['detail']}]"
        a = agg.setdefault(key, {"launches": 0, "ncu_ms": 0.0, "dram_read": 0.0, "dram_write": 0.0,
                                 "algo_bytes": 0.0, "flops": 0.0, "kernel": name.split("(")[0]})
        a["launches"] += 1
        a["ncu_ms"] += m.get("gpu__time_duration.sum", 0.0) / 1e6
        a["dram_read"] += m.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += m.get("dram__bytes_write.sum", 0.0)
        a["algo_bytes"] += r["algo_bytes"] or 0.0
        a["flops"] += r["flops"]
    res = OrderedDict()
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ncu_ms"]):
        n = a["launches"]
        dram = (a["dram_read"] + a["dram_write"]) / n
        res[k] = {"kernel": a["kernel"], "launches": n, "ncu_ms_per_launch": round(a["ncu_ms"] / n, 4),
                  "dram_read_gb_per_launch": round(a["dram_read"] / n / 1e9, 4),
                  "dram_write_gb_per_launch": round(a["dram_write"] / n / 1e9, 4),
                  "algo_gb_per_launch": round(a["algo_bytes"] / n / 1e9, 4),
                  "dram_over_algo": round(dram / (a["algo_bytes"] / n), 3) if a["algo_bytes"] else None,
                  "dram_gbs": round(dram / (a["ncu_ms"] / n / 1e3) / 1e9, 1) if a["ncu_ms"] else None,
                  "tflops": round(a["flops"] / (a["ncu_ms"] / 1e3) / 1e12, 1) if a["ncu_ms"] and a["flops"] else None}
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        print(f"{k:48s} {v['launches']:5d} {v['ncu_ms_per_launch']:9.3f} ms  dram {v['dram_read_gb_per_launch'] + v['dram_write_gb_per_launch']:7.3f} GB"
              f"  algo {v['algo_gb_per_launch']:7.3f} GB  x{v['dram_over_algo']}")
    if traffic_out:
        gemms = {k: v for k, v in res.items() if k.startswith("gemm[")}
        dom = max(gemms.items(), key=lambda kv: kv[1]["ncu_ms_per_launch"] * kv[1]["launches"])
        json.dump({"shape": dom[0], "kernel": dom[1]["kernel"],
                   "dram_bytes_per_launch": (dom[1]["dram_read_gb_per_launch"] + dom[1]["dram_write_gb_per_launch"]) * 1e9,
                   "algo_bytes_per_launch": dom[1]["algo_gb_per_launch"] * 1e9,
                   "dram_over_algo": dom[1]["dram_over_algo"], "source": lpath}, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
