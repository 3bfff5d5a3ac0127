#!/bin/bash
# Raster-order experiment: per-launch duration (base clocks) and DRAM bytes of the pair GEMM
# for several PLORA_PAIR_BAND settings on the gemm_once shapes.
for b in 0 4 16 32 -4 -8 -16; do
  PLORA_PAIR_BAND=$b ncu --clock-control base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:plora_gemm_pair --csv python tools/gemm_once.py 2>/dev/null | grep -E "gpu__time|dram__bytes" \
    | awk -F'","' -v b=$b '{gsub(/"/,"",$NF); print b, $(NF-2), $NF}'
done
