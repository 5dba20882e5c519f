"""Per-launch summary of an `ncu --metrics ... --csv` capture: time, DRAM read/write."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [k for k, line in enumerate(lines) if line.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ki, mi, vi, gi = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Grid Size"))
agg = collections.OrderedDict()
for r in rows[1:]:
    agg.setdefault((r[0], r[ki].split("(")[0][-44:], r[gi]), {})[r[mi]] = float(r[vi].replace(",", ""))
for (i, k, g), m in agg.items():
    print(f"{i:>3} {k:<46} {g:<14} t={m.get('gpu__time_duration.sum', 0) / 1e3:9.1f}us "
          f"rd={m.get('dram__bytes_read.sum', 0) / 1e9:7.2f}GB wr={m.get('dram__bytes_write.sum', 0) / 1e9:6.2f}GB")
