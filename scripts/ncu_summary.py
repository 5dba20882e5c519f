"""Summarise ncu captures brought back in gpurun_out/ into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/hist_r01 [--launches gpurun_out/launches.csv]

Writes <out>.txt (key metrics per kernel) and merges the per-launch DRAM
traffic (dram__bytes_read.sum + dram__bytes_write.sum) into
profiles/traffic.json, which bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_static",
    "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__cycles_elapsed.avg.per_second",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel\w*)", name)
    return m.group(1) if m else name[:60]


def raw(rep: str) -> list[dict]:
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def to_bytes(d: dict, key: str) -> float:
    v = float(d[key].replace(",", ""))
    return v * UNIT.get(d["_units"].get(key, "byte"), 1)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    lines = []
    traffic_path = Path("profiles/traffic.json")
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for d in raw(a.rep):
        name = short(d["Kernel Name"])
        lines.append(f"== {d['Kernel Name']}")
        for k in KEYS:
            if k in d:
                lines.append(f"   {k:60s} {d[k]:>16s} {d['_units'].get(k, '')}")
        t = to_bytes(d, "dram__bytes_read.sum") + to_bytes(d, "dram__bytes_write.sum")
        lines.append(f"   dram traffic per launch (read+write)                         {t:16.0f} byte")
        traffic[name] = t
    if a.launches:
        tot = defaultdict(float)
        cnt = defaultdict(int)
        text = Path(a.launches).read_text()
        body = text[text.index('"ID"'):]
        for r in csv.DictReader(io.StringIO(body)):
            if r.get("Metric Name") == "gpu__time_duration.sum":
                n = short(r["Kernel Name"])
                tot[n] += float(r["Metric Value"].replace(",", ""))
                cnt[n] += 1
        all_ns = sum(tot.values())
        lines.append("\n== launch list (ncu gpu__time_duration.sum, cold-cache, serialised)")
        for n in sorted(tot, key=lambda k: -tot[k]):
            lines.append(f"   {n:50s} launches={cnt[n]:4d} total_us={tot[n] / 1e3:10.1f} share={tot[n] / all_ns:6.1%}")
    Path(a.out + ".txt").write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
