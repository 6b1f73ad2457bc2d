"""Developer tool: top stall sites of one kernel from an ncu report's
source page (ncu -i REP --page source --csv --print-source sass)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# one section per captured kernel instance: "Kernel Name" line, header, rows
data, hdr = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is not None and len(r) == len(hdr):
        data.append(r)
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {h: sum(float(r[ix[h]] or 0) for r in data) for h in reasons}
print(f"samples {tot:.0f}")
print("  ".join(f"{h[6:]} {v / tot * 100:.1f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
for r in sorted(data, key=lambda r: -float(r[ix[S]] or 0))[:n]:
    s = float(r[ix[S]] or 0)
    det = sorted(((float(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{r[0][-5:]:>6s} {s / tot * 100:5.2f}% {r[1][:58]:58s} " + " ".join(f"{d[1]}:{d[0]:.0f}" for d in det))
