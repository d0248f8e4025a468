#!/usr/bin/env python
"""Collect a tools/final_r02.sh run into profiles/: bench lines, e2e log,
launch list, ncu --set full summaries and the per-iteration DRAM traffic.

    python tools/collect_final.py gpurun_out/final_r02b profiles/r02/final
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

SRC, DST = sys.argv[1], sys.argv[2]
os.makedirs(DST, exist_ok=True)
HERE = os.path.dirname(os.path.abspath(__file__))


def last_json(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        return None


rows = []
for name in ("c1", "c2", "c3", "c4", "c5", "reference_arm"):
    d = last_json(os.path.join(SRC, f"bench_{name}.json"))
    if d is None:
        print(f"bench_{name}: missing or empty (kept the previous copy)")
        continue
    shutil.copy(os.path.join(SRC, f"bench_{name}.json"), DST)
    r, e, c = d.get("roofline") or {}, d.get("e2e") or {}, d.get("clocks") or {}
    rows.append((name, d["value"], d["ms_per_step"], e.get("value"), r.get("kernel"), r.get("frac"),
                 r.get("iteration_frac"), c.get("sm_mhz"), c.get("reasons"),
                 (d.get("cpu_baseline") or {}).get("value")))
for r in rows:
    print(" ".join(str(x) if not isinstance(x, float) else "%.4g" % x for x in r))

for f in ("e2e.log", "smi.txt", "launches_c2.csv"):
    if os.path.exists(os.path.join(SRC, f)):
        shutil.copy(os.path.join(SRC, f), DST)


def summary(args, out):
    r = subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), *args], capture_output=True, text=True)
    if r.returncode == 0:
        open(os.path.join(DST, out), "w").write(r.stdout)
    else:
        print("ncu_summary failed:", args, r.stderr[-300:])


if os.path.exists(os.path.join(SRC, "launches_c2.csv")):
    summary(["--launches", os.path.join(SRC, "launches_c2.csv")], "launches_c2.md")
for rep, out in (("prof_x.ncu-rep", "ncu_full_c2_xpass.md"), ("prof_yz.ncu-rep", "ncu_full_c2_yz.md")):
    if os.path.exists(os.path.join(SRC, rep)):
        summary([os.path.join(SRC, rep)], out)


def iter_traffic(path):
    """DRAM bytes and kernel time per RL iteration from an ncu --metrics CSV:
    only whole iterations are counted, from the first x-pass launch of the
    window to the last one that starts an iteration (2 x passes each)."""
    txt = open(path).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    ids = []
    for row in rows:
        if row["ID"] not in ids:
            ids.append(row["ID"])
    name = {row["ID"]: row["Kernel Name"] for row in rows}
    xs = [i for i in ids if "xpass" in name[i]]
    iters = (len(xs) - 1) // 2
    if iters < 1:
        return None, 0, 0, 0
    keep = set(ids[ids.index(xs[0]):ids.index(xs[2 * iters])])
    acc = collections.defaultdict(float)
    for row in rows:
        if row["ID"] not in keep:
            continue
        k = row["Kernel Name"]
        kind = "x" if "xpass" in k else "y" if "ypass" in k else "z"
        v = float(row["Metric Value"].replace(",", ""))
        unit = row["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                 "msecond": 1}.get(unit, 1)
        acc[(kind, row["Metric Name"])] += v * scale
    out = {}
    for kind in "xyz":
        out[kind] = (acc[(kind, "dram__bytes_read.sum")] / iters / 1e6, acc[(kind, "dram__bytes_write.sum")] / iters / 1e6)
    tot = sum(a + b for a, b in out.values()) / 1e3
    t = sum(v for (k, m), v in acc.items() if m == "gpu__time_duration.sum") / iters
    return out, tot, t, iters


lines = []
for f, label in (("iter.csv", "kx-chunked y/z (default)"), ("iter_whole.csv", "whole-volume passes (`VK_RL_KXCHUNK=0`)")):
    p = os.path.join(SRC, f)
    if not os.path.exists(p):
        continue
    out, tot, t, iters = iter_traffic(p)
    if out is None:
        print(f"{f}: fewer than one whole iteration in the window")
        continue
    lines.append(f"| {label} | {out['x'][0]:.0f} / {out['x'][1]:.0f} MB | {out['y'][0]:.0f} / {out['y'][1]:.0f} MB | "
                 f"{out['z'][0]:.0f} / {out['z'][1]:.0f} MB | **{tot:.2f} GB** | {t:.3f} ms | {iters} |")
if lines:
    with open(os.path.join(DST, "iteration_traffic_table.md"), "w") as f:
        f.write("| schedule | x pass R / W | y passes R / W | z passes R / W | DRAM per iteration | serialised kernel time | iterations averaged |\n")
        f.write("|---|---|---|---|---|---|---|\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))
