"""Summarise ncu outputs into committed profiles/ artifacts (dev tool).

  python bench_tools/ncu_summarize.py full   <report.ncu-rep> <out.json>
      per kernel (first captured launch of each name): duration, dram bytes
      read/write per launch, tensor-pipe / dram / sm throughput, registers.
  python bench_tools/ncu_summarize.py launches <launches.csv> <out.txt>
      the --metrics gpu__time_duration.sum launch list -> per-kernel count,
      total time and share of the captured step.
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}


def short(name):
    m = re.search(r"(ttt_\w+?)(?:<|\(|$)", name)
    return m.group(1) if m else name.split("(")[0]


def full(rep, out):
    txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = OrderedDict()
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        if name in res:
            continue
        d = {}
        for m, key in FULL_METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            v *= SCALE.get(units[i], 1.0)
            d[key] = v
        if "dram_read" in d and "dram_write" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d["dram_write"]
        d["duration_note"] = "ncu replay (clock-control as captured); compare shares, not absolutes"
        res[name] = d
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


def launches(csvf, out):
    rows = list(csv.reader(open(csvf)))
    # find header row
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    kn, mn, mv, mu = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = short(r[kn])
        v = float(r[mv].replace(",", "")) * SCALE.get(r[mu], 1e-9)
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + v)
    ours = {k: v for k, v in agg.items() if k.startswith("ttt_")}
    tot = sum(t for _, t in ours.values())
    lines = [f"{'kernel (this library; share of their total)':44s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>9s} {'share':>7s}"]
    for name, (c, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name:44s} {c:8d} {t * 1e3:10.3f} {t / c * 1e6:9.1f} {t / tot:7.1%}")
    lines.append(f"{'TOTAL':44s} {sum(c for c, _ in ours.values()):8d} {tot * 1e3:10.3f}")
    other = {k: v for k, v in agg.items() if not k.startswith("ttt_")}
    if other:
        lines.append("other kernels in the captured process (input generation / buffer zeroing at setup, not in the step):")
        for name, (c, t) in sorted(other.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"  {name[:80]:80s} {c:5d} {t * 1e3:9.3f} ms")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
