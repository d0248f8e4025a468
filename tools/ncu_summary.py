#!/usr/bin/env python
"""Summarise an ncu report (raw page) or an ncu launch-list CSV into profiles/.

    python tools/ncu_summary.py report.ncu-rep > profiles/rNN/xxx.md
    python tools/ncu_summary.py --launches launches.csv > profiles/rNN/launches.md
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    print(f"# ncu --set full summary: `{path}`\n")
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in data:
        cells = []
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                cells.append(f"{r[i]} {units[i]}".strip())
            else:
                cells.append("-")
        print(f"| {r[h.index('Kernel Name')][:40]} | " + " | ".join(cells) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k = r[ki].split("(")[0]
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    print(f"# ncu launch list (gpu__time_duration.sum, cold-cache, serialised): `{path}`\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / cnt[k]:.1f} | {tot[k] / s:.3f} |")


if __name__ == "__main__" and sys.argv[1] != "--source":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])


def source_hotspots(path, kernel_regex, top=25):
    """Per CUDA source line: warp-instructions executed and stall samples
    (needs a capture with --import-source on and -lineinfo)."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "-k", f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows, cur_file, header = [], None, None
    for r in csv.reader(io.StringIO(raw)):
        if len(r) == 2 and r[0] in ("File Path", "File Name"):
            cur_file = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            header = r
        elif header and len(r) == len(header) and r[0].isdigit() and r[2] == "-":
            d = dict(zip(header, r))
            def num(k):
                try:
                    return float(d.get(k, "0").replace(",", ""))
                except ValueError:
                    return 0.0
            stalls = {k: num(k) for k in header if k.startswith("stall_") and "Not Issued" not in k}
            rows.append((cur_file, int(r[0]), r[1].strip()[:70], num("Instructions Executed"),
                         num("Warp Stall Sampling (All Samples)"), stalls))
    tot_i = sum(x[3] for x in rows) or 1
    tot_s = sum(x[4] for x in rows) or 1
    print(f"# source hotspots `{path}` kernel~{kernel_regex}: {tot_i:.3g} warp-instr, {tot_s:.0f} stall samples\n")
    print("| file:line | instr % | stall % | top stalls | source |")
    print("|---|---|---|---|---|")
    for f, ln, src, ins, st, stalls in sorted(rows, key=lambda x: -x[4])[:top]:
        ts = ", ".join(f"{k[6:]}={v:.0f}" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"| {f}:{ln} | {100 * ins / tot_i:.1f} | {100 * st / tot_s:.1f} | {ts} | `{src}` |")


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[1] == "--source":
    source_hotspots(sys.argv[2], sys.argv[3])
