"""Developer tool: table of tools/variant_probe.sh results (gpurun_out/vp_*.csv)."""
import csv, glob, os, sys
for f in sorted(glob.glob("gpurun_out/vp_*.csv")):
    rows = list(csv.DictReader(open(f)))
    by = {}
    for r in rows:
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        by.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
    for k, m in by.items():
        print(f"{os.path.basename(f)[3:-4]:22s} {k:18s} t={float(m['gpu__time_duration.sum'])/1e6:8.3f} ms"
              f" cyc={float(m['sm__cycles_elapsed.max'])/1e6:8.2f}M clk={float(m['sm__cycles_elapsed.avg.per_second'])/1e9:.2f}G"
              f" tensor={m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']}% issue={m['sm__issue_active.avg.pct_of_peak_sustained_elapsed']}%"
              f" inst={float(m['smsp__inst_executed.sum'])/1e6:.0f}M")
