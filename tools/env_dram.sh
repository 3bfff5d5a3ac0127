#!/bin/bash
# DRAM bytes + duration of the first 8 pair-GEMM launches of a C3 step (layer 0-1 forward:
# qkv group, o, gate/up+SwiGLU, down) under environment settings given as arguments, e.g.
#   tools/env_dram.sh PLORA_DEBUG_FLAGS=0 PLORA_DEBUG_FLAGS=144
mkdir -p gpurun_out
for kv in "$@"; do
  tag=$(echo "$kv" | tr '=' '_')
  env "$kv" timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:plora_gemm_pair -c 8 --csv --log-file gpurun_out/envdram_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$tag" <<'PY'
import csv, sys, collections
tag = sys.argv[1]
conv = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3,
        'ns': 1e-9, 'nsecond': 1e-9}
per = collections.defaultdict(dict)
for r in csv.reader(open(f"gpurun_out/envdram_{tag}.csv")):
    if len(r) > 14 and r[0].isdigit():
        per[int(r[0])][r[12]] = float(r[14].replace(',', '')) * conv[r[13]]
for i, d in sorted(per.items()):
    print(f"{tag} launch {i}: rd {d['dram__bytes_read.sum']/1e6:7.0f} MB wr {d['dram__bytes_write.sum']/1e6:6.0f} MB "
          f"t {d['gpu__time_duration.sum']*1e6:7.0f} us")
PY
done
