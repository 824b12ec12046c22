"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

    python tools/ncu_summary.py report  gpurun_out/prof.ncu-rep  profiles/r01_k1.md
    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python tools/ncu_summary.py traffic gpurun_out/prof.ncu-rep ax_tma_kernel profiles/k1_traffic.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1,
         "msecond": 1e-3, "second": 1}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def val(hdr, units, row, key):
    if key not in hdr:
        return None, ""
    i = hdr.index(key)
    try:
        return float(row[i].replace(",", "")), units[i]
    except ValueError:
        return None, units[i]


def report(rep, dst):
    hdr, units, rows = raw_rows(rep)
    lines = [f"# ncu summary of `{rep}`", ""]
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        lines.append(f"## `{name[:160]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        t, tu = val(hdr, units, r, "gpu__time_duration.sum")
        rd, ru = val(hdr, units, r, "dram__bytes_read.sum")
        wr, wu = val(hdr, units, r, "dram__bytes_write.sum")
        for key, label in KEYS:
            v, u = val(hdr, units, r, key)
            if v is not None:
                lines.append(f"| {label} (`{key}`) | {v:,.3f} {u} |")
        if t and rd is not None and wr is not None:
            secs = t * SCALE.get(tu, 1e-9)
            tot = rd * SCALE.get(ru, 1) + wr * SCALE.get(wu, 1)
            lines.append(f"| DRAM bytes / duration | {tot / secs / 1e9:,.1f} GB/s |")
        stalls = []
        for h, v in zip(hdr, r):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(v.replace(",", "")), h.split("stalled_")[1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot_s = sum(s for s, _ in stalls) or 1
        lines.append("")
        lines.append("Top warp stall reasons (pc sampling): " +
                     ", ".join(f"{n} {100 * s / tot_s:.0f}%" for s, n in stalls[:5]))
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def traffic(rep, pattern, dst):
    hdr, units, rows = raw_rows(rep)
    out = []
    for r in rows:
        name = r[hdr.index("Kernel Name")]
        if pattern not in name:
            continue
        rd, ru = val(hdr, units, r, "dram__bytes_read.sum")
        wr, wu = val(hdr, units, r, "dram__bytes_write.sum")
        out.append(rd * SCALE.get(ru, 1) + wr * SCALE.get(wu, 1))
    res = {"kernel": pattern, "bytes_per_launch": sum(out) / len(out) if out else None,
           "launches": len(out), "source": rep}
    json.dump(res, open(dst, "w"), indent=1)
    print(res)


def launches(src, dst):
    per = defaultdict(lambda: [0, 0.0])
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    for r in rows[start + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        short = r[ki].split("(")[0][:90]
        per[short][0] += 1
        per[short][1] += v
    tot = sum(v[1] for v in per.values()) or 1
    lines = [f"# launch list `{src}` (ncu, cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t * 1e3:.3f} | {t / c * 1e6:.1f} | {100 * t / tot:.1f}% |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "report":
        report(sys.argv[2], sys.argv[3])
    elif mode == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
