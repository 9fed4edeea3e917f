"""Top SASS instructions by stall samples from an ncu report: python tools/ncu_sass.py rep.ncu-rep <kernel regex> [top] [launch id]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}"] +
                     (["--launch-skip", sys.argv[4], "--launch-count", "1"] if len(sys.argv) > 4 else []),
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
items = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        items.append((int(d.get("# Samples", d.get("Warp Stall Sampling (All Samples)", "0")) or 0), d))
    except ValueError:
        pass
if not items:
    print(hdr)
    sys.exit()
tot = sum(s for s, _ in items) or 1
idx = {id(d): i for i, (_, d) in enumerate(items)}
print("total samples", tot, "columns:", [h for h in hdr if "stall" in h.lower()][:3])
for s, d in sorted(items, key=lambda x: -x[0])[:top]:
    why = sorted(((int(d[h] or 0), h) for h in hdr if h.startswith("stall_") and d.get(h) not in ("", "0", None)), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}%  #{idx[id(d)]:5d} {d['Source'][:70]:70}  inst={d.get('# Instructions Executed', d.get('Instructions Executed',''))}  {[(h[6:],v) for v,h in why]}")
