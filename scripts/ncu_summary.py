"""Summarise ncu reports / launch lists into text files for profiles/.

python scripts/ncu_summary.py report  <file.ncu-rep> <out.txt>
python scripts/ncu_summary.py launches <launches.csv> <out.txt>
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "smsp__inst_executed.sum",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def report(path, out):
    raw = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "raw", "--csv"))))
    h, units = raw[0], raw[1]
    lines = [f"# ncu --set full summary of {path}", ""]
    for r in raw[2:]:
        lines.append(f"## {r[h.index('Kernel Name')]}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"  {m:60s} {r[i]:>16s} {units[i]}")
        lines.append("")
    src = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "source", "--csv"))))
    if len(src) > 2:
        hh = src[1]
        cols = [i for i, n in enumerate(hh) if n.startswith("stall_") and "Not Issued" not in n]
        tot = collections.Counter()
        for r in src[2:]:
            if len(r) > max(cols):
                tot.update({hh[i]: int(r[i]) for i in cols if r[i].isdigit()})
        s = sum(tot.values()) or 1
        lines.append("## warp stall samples (first kernel in report)")
        for k, v in tot.most_common(10):
            lines.append(f"  {k:30s} {v:7d} {100 * v / s:5.1f}%")
    open(out, "w").write("\n".join(lines) + "\n")


_SCALE = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0, "": 1.0, "inst": 1.0}


def launches(path, out):
    """Per-kernel means of a `ncu --metrics ... --csv` launch list (times in ns,
    bytes in B whatever unit ncu chose; 'n/a' entries skipped)."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[hi + 1:]:
        if len(r) > vi:
            try:
                v = float(r[vi].replace(",", ""))
            except ValueError:
                continue
            if ui is not None:
                v *= _SCALE.get(r[ui], 1.0)
            agg[r[ki][:90]][r[mi]].append(v)
    tot = sum(sum(d["gpu__time_duration.sum"]) for d in agg.values()) or 1
    extra = sorted({m for d in agg.values() for m in d} - {"gpu__time_duration.sum", "dram__bytes_read.sum",
                                                           "dram__bytes_write.sum"})
    lines = [f"# per-kernel launch list summary of {path} (cold-cache, serialised by ncu)", "",
             f"{'kernel':90s} {'n':>4s} {'mean_us':>9s} {'share':>6s} {'dramR_MB':>9s} {'dramW_MB':>9s}"
             + "".join(f" {m[:28]:>28s}" for m in extra)]
    for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        t = d["gpu__time_duration.sum"]
        if not t:
            continue
        rd = d.get("dram__bytes_read.sum") or [0]
        wr = d.get("dram__bytes_write.sum") or [0]
        lines.append(f"{k:90s} {len(t):4d} {sum(t) / len(t) / 1e3:9.2f} {100 * sum(t) / tot:5.1f}% "
                     f"{sum(rd) / len(rd) / 1e6:9.1f} {sum(wr) / len(wr) / 1e6:9.1f}"
                     + "".join(f" {sum(d[m]) / len(d[m]) if d.get(m) else float('nan'):28.2f}" for m in extra))
    lines.append(f"\n# total device time of the listed launches: {tot / 1e3:.1f} us")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
