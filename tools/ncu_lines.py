"""Stall samples and executed instructions aggregated per CUDA source line from an ncu report
(--print-source cuda,sass; needs -lineinfo):  python tools/ncu_lines.py rep.ncu-rep <kernel regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
f = None
hdr = None
agg = collections.defaultdict(lambda: [0, 0, "", collections.Counter()])
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        hdr = None
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:  # a source line row: remember it, SASS rows follow with empty line number
        line = (f, r[0])
        agg[line][2] = r[1].strip()[:90]
        continue
    try:
        agg[line][0] += int(r[4] or 0)
        agg[line][1] += int(r[7] or 0)
        for j, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name and r[j] not in ("", "0"):
                agg[line][3][name[6:]] += int(r[j])
    except (ValueError, IndexError, NameError):
        pass
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"samples {tot_s}  warp instructions {tot_i}")
for (fn, ln), (s, i, src, why) in sorted(agg.items(), key=lambda kv: -kv[1][1 if "--by-inst" in sys.argv else 0])[:top]:
    reasons = " ".join(f"{k}:{100 * v / max(s, 1):.0f}" for k, v in why.most_common(3))
    print(f"{100 * s / tot_s:5.1f}% stall {100 * i / tot_i:5.1f}% inst  {fn}:{ln:>4}  {src[:60]:60}  [{reasons}]")
