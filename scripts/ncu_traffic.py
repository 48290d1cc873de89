"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) from ncu
--set full captures -> profiles/traffic_rNN.json (NN from $VOX_ROUND, default 02) ({kernel class: bytes per launch}),
plus a one-line-per-launch summary of the key counters.

usage: python scripts/ncu_traffic.py gemm=gpurun_out/prof_gemm.ncu-rep attn=gpurun_out/prof_attn.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0], "grid": r[h.index("Grid Size")]}
        for k in KEYS:
            if k in h:
                v = float(r[h.index(k)].replace(",", ""))
                u = units[h.index(k)]
                d[k] = v * UNIT.get(u, 1) if "bytes" in k else v
        yield d


def main():
    res = {}
    lines = []
    for arg in sys.argv[1:]:
        cls, rep = arg.split("=", 1)
        launches = list(rows_of(rep))
        tot = [l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in launches]
        res[cls] = round(sum(tot) / len(tot))
        for l in launches:
            lines.append(f"{cls:6s} {l['kernel'][:40]:40s} grid {l['grid']:14s} "
                         f"{l['gpu__time_duration.sum']:8.2f} us  dram {(l['dram__bytes_read.sum'] + l['dram__bytes_write.sum']) / 1e6:8.2f} MB  "
                         f"dram% {l.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}  "
                         f"tensor% {l.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):5.1f}  "
                         f"lts% {l.get('lts__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}  "
                         f"regs {int(l.get('launch__registers_per_thread', 0))}")
    import os
    rnd = os.environ.get("VOX_ROUND", "02")
    (ROOT / "profiles" / f"traffic_r{rnd}.json").write_text(json.dumps(res, indent=1) + "\n")
    print("\n".join(lines))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
