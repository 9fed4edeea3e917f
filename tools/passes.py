"""One-line pass summary of bench.py JSON lines (A/B runs):  python tools/passes.py tag < bench.json"""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "passes" not in d:
        print(tag, line[:200])
        continue
    ps = " | ".join(f"{p['role'][0]}:{p['scheme']} {p['ms']:.3f}ms {p['frac_hbm']:.2f}" for p in d["passes"])
    print(f"{tag:12s} {d['value'] / 1e9:7.2f} G/s {d['ms_per_step']:.3f} ms/step  {ps}  parity={d.get('parity', {}).get('max_rel_err')}")
