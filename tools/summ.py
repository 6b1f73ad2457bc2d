"""Developer tool: one-line summaries of bench JSON lines (files or jsonl)."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        try:
            d = json.loads(line)
        except Exception:
            continue
        rs = d.get("roofline_stages", {})
        st = " ".join(f"{k}={v['ms']:.3f}({v['frac']:.2f})" for k, v in rs.items())
        lay = d.get("config", {}).get("layer")
        lay = lay.get("name") if isinstance(lay, dict) else lay
        print(f"{f.split('/')[-1]} {lay or ''} {d.get('ms_per_step', 0):.3f}ms {d.get('value', 0):.3g} {st}")
