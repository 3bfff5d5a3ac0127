"""Key counters per launch from an .ncu-rep (duration, DRAM bytes/throughput, SM balance)."""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "sm__cycles_active.max",
        "sm__cycles_active.min", "gpc__cycles_elapsed.max", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "launch__grid_size", "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print("---")
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w}: {r[i]} {units[i]}")
