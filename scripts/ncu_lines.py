"""Per-source-line stall samples and instruction counts from an ncu report
(compile with -lineinfo):  python scripts/ncu_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0] or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        i = int(d["Instructions Executed"] or 0)
    except ValueError:
        continue
    top_stalls = sorted(((k, float(v or 0)) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                         and v not in ("", "-")), key=lambda kv: -kv[1])[:3]
    out.append((s, int(r[0]), i, r[1].strip()[:70], top_stalls))
tot = sum(o[0] for o in out) or 1
for s, ln, i, src, st in sorted(out, key=lambda o: -o[0])[:top]:
    sts = " ".join(f"{k[6:]}:{int(v)}" for k, v in st if v)
    print(f"{ln:5d} {100 * s / tot:5.1f}% inst={i:11d} {src:70s} {sts}")
