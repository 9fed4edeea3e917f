"""One-screen summary of a bench.py JSON line: python tools/bench_brief.py gpurun_out/bench.json"""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print(f"value {d.get('value', 0) / 1e9:.2f} G/s  ms/step {d.get('ms_per_step', 0):.3f}  n_gpus {d.get('n_gpus')}  "
          f"clocks {d.get('clocks')}")
    r = d.get("roofline", {})
    print(f"roofline {r.get('kernel')} {r.get('achieved')} GB/s frac {r.get('frac')} frac_8tbs {r.get('frac_8tbs')} "
          f"traffic {r.get('traffic')}")
    for p in d.get("passes", []):
        print("  ", {k: p[k] for k in p if k not in ("alg_bytes",)})
    for key in ("step_frac_hbm", "step_frac_8tbs", "e2e", "parity", "cpu_baseline", "exchange", "same_level",
                "nonfinite_flag", "setup_s", "gpu_launches"):
        if key in d:
            v = d[key]
            if isinstance(v, dict):
                v = {a: b for a, b in v.items() if a not in ("how", "sample")}
            print(f"{key}: {v}")
