"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
k = 0
while k < len(rows):
    if rows[k] and rows[k][0] == "Kernel Name":
        name = rows[k][1]
        hdr = rows[k + 1]
        si, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
        items, j = [], k + 2
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            try:
                items.append((int(rows[j][si]), j - k - 2, rows[j][src].strip()))
            except (ValueError, IndexError):
                pass
            j += 1
        tot = sum(i[0] for i in items)
        print(f"== {name}  total samples {tot}")
        for n, idx, s in sorted(items, reverse=True)[:top]:
            print(f"{n:7d} {100*n/max(tot,1):5.1f}%  #{idx:5d}  {s[:100]}")
        k = j
    else:
        k += 1
