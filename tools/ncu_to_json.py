"""Condense an .ncu-rep into a small JSON of the counters DESIGN.md / bench.py cite:
per launch duration, DRAM bytes and throughput, L2->SMEM TMA bytes, tensor-memory pipe
activity, SM balance.  Usage: python tools/ncu_to_json.py rep.ncu-rep out.json [note]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "kernel": "Kernel Name",
    "duration_us": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tma_l2_to_smem_bytes": "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "tensor_mem_pipe_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "sm_cycles_active_avg": "sm__cycles_active.avg",
    "sm_cycles_active_max": "sm__cycles_active.max",
    "sm_cycles_active_min": "sm__cycles_active.min",
    "gpc_cycles_elapsed_max": "gpc__cycles_elapsed.max",
    "gpc_clock_ghz": "gpc__cycles_elapsed.max.per_second",
    "registers_per_thread": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "nsecond": 1e-3, "ns": 1e-3, "Tbyte": 1e12}

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    d = {}
    for k, col in KEYS.items():
        if col not in hdr:
            continue
        i = hdr.index(col)
        v, u = r[i], units[i]
        if k == "kernel":
            d[k] = v
            continue
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            d[k] = v
            continue
        if "bytes" in k:
            x *= SCALE.get(u, 1.0)
        if k == "duration_us" and u in SCALE:
            x *= SCALE[u]
        d[k] = round(x, 4)
    if "dram_bytes_read" in d and "dram_bytes_write" in d:
        d["dram_bytes"] = d["dram_bytes_read"] + d["dram_bytes_write"]
        d["dram_gbs"] = round(d["dram_bytes"] / (d["duration_us"] * 1e3), 1)
    out.append(d)
doc = {"source": f"ncu --set full --clock-control none ({sys.argv[1].split('/')[-1]})", "launches": out}
if len(sys.argv) > 3:
    doc["note"] = sys.argv[3]
json.dump(doc, open(sys.argv[2], "w"), indent=1)
print(json.dumps(doc, indent=1)[:3000])
