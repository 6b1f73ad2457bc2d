"""Developer tool: table of tools/stub_sweep.sh results."""
import json
import sys

for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/stub_sweep.jsonl"):
    try:
        d = json.loads(line)
    except ValueError:
        print("bad line", line[:80])
        continue
    b = d["line"]
    st = b["roofline_stages"]
    print(f"{d['variant'] or 'full':8s} {d['cfg']:8s} L{d['layer']:<2d} step {b['ms_per_step']:.3f}  "
          + "  ".join(f"{k} {v['ms']:.3f}" for k, v in st.items()))
