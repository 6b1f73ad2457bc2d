#!/usr/bin/env python3
"""Summarise a round's ncu captures into profiles/ (run here, no GPU).

  python tools/ncu_summary.py <launches.csv> <prof.ncu-rep> <config-name> <round>

Writes profiles/<round>_<config>_launches.md (share of device time per kernel
over the timed steps of the launch list), profiles/<round>_<config>_full.md
(per-kernel metrics of the --set full capture) and
profiles/traffic_<config>.json (dram bytes read+write per launch, keyed by
bench stage, read by bench.py for roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = {"k_fwd_tc": "fwd_vmm", "k_bwd_tc": "bwd_vmm", "k_dw_tc": "dw", "k_dw": "dw", "k_update4": "update", "k_update": "update", "k_update_tma": "update",
         "k_prep_x": "prep_x", "k_prep_dy": "prep_dy"}
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name):
    n = name.split("(")[0].split("<")[0].strip()
    return n.split()[-1].split("::")[-1]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r["Metric Name"] == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1)))
    return rows


def full(path):
    # an .ncu-rep, or its `ncu -i REP --page raw --csv` export
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    hdr = next(csv.reader([lines[0]]))
    units = next(csv.reader([lines[1]]))
    res = []
    for ln in lines[2:]:
        v = next(csv.reader([ln]))
        d = dict(zip(hdr, v))
        u = dict(zip(hdr, units))
        res.append((short(d["Kernel Name"]), d, u))
    return res


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)


def main():
    lpath, rpath, cfg, rnd = sys.argv[1:5]
    prof = os.path.join(ROOT, "profiles")
    L = launches(lpath)
    # timed region = everything after the last create-time kernel; report the
    # per-step kernels only (the launch list covers warm-up + 2 timed steps)
    per = collections.defaultdict(lambda: [0.0, 0])
    for k, us in L:
        per[k][0] += us
        per[k][1] += 1
    step_kernels = {k: v for k, v in per.items() if k in STAGE or k.startswith("k_absmax")}
    tot = sum(v[0] for v in step_kernels.values())
    with open(os.path.join(prof, f"{rnd}_{cfg}_launches.md"), "w") as f:
        f.write(f"# ncu launch list, {cfg} ({rnd})\n\n`{os.path.basename(lpath)}`: `ncu --metrics gpu__time_duration.sum "
                "--clock-control none` over `bench.py --steps 2 --warmup 3` (5 steps + core creation). Cold-cache and "
                "serialised: compare shares, not absolutes.\n\n| kernel | launches | total us | avg us | share of per-step "
                "kernels |\n|---|---|---|---|---|\n")
        for k, (us, n) in sorted(per.items(), key=lambda kv: -kv[1][0]):
            share = f"{100 * us / tot:.1f}%" if k in step_kernels else "(create-time)"
            f.write(f"| {k} | {n} | {us:.1f} | {us / n:.1f} | {share} |\n")
    F = full(rpath)
    traffic = {}
    with open(os.path.join(prof, f"{rnd}_{cfg}_full.md"), "w") as f:
        f.write(f"# ncu --set full, {cfg} ({rnd})\n\nOne launch of each per-step kernel after 3 warm-up steps "
                "(`tools/profile_round.sh`).\n\n| kernel | " + " | ".join(m[1] for m in METRICS) + " |\n|---|" +
                "---|" * len(METRICS) + "\n")
        for k, d, u in F:
            cells = []
            for m, _ in METRICS:
                cells.append(f"{d.get(m, '')} {u.get(m, '')}".strip())
            f.write(f"| {k} | " + " | ".join(cells) + " |\n")
            st = STAGE.get(k)
            if st and "dram__bytes_read.sum" in d:
                t = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + to_bytes(
                    d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
                traffic[st] = t if t == t else None  # a metric ncu could not collect reads nan
    traffic["source"] = f"profiles/{rnd}_{cfg}_full.md (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    with open(os.path.join(prof, f"traffic_{cfg}.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print(open(os.path.join(prof, f"{rnd}_{cfg}_full.md")).read())
    print(open(os.path.join(prof, f"{rnd}_{cfg}_launches.md")).read())


if __name__ == "__main__":
    main()
