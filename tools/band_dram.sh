#!/bin/bash
# DRAM bytes per pair-GEMM launch of one C3 layer (forward + backward) under several
# N-band widths (PLORA_PAIR_BAND), one ncu pass each.  Usage: tools/band_dram.sh -8 -16 ...
mkdir -p gpurun_out
for b in "$@"; do
  PLORA_PAIR_BAND=$b timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:plora_gemm_pair -c 8 --csv --log-file gpurun_out/band_$b.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  python - "$b" <<'PY'
import csv, sys, collections
b = sys.argv[1]
conv = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3,
        'ns': 1e-9, 'nsecond': 1e-9}
per = collections.defaultdict(dict)
for r in csv.reader(open(f"gpurun_out/band_{b}.csv")):
    if len(r) > 14 and r[0].isdigit():
        per[int(r[0])][r[12]] = float(r[14].replace(',', '')) * conv[r[13]]
for i, d in sorted(per.items()):
    print(f"band {b} launch {i}: rd {d['dram__bytes_read.sum']/1e6:7.0f} MB wr {d['dram__bytes_write.sum']/1e6:6.0f} MB "
          f"t {d['gpu__time_duration.sum']*1e6:7.0f} us")
PY
done
