"""Summaries for profiles/ from ncu outputs brought back by gpurun.

  python tools/summarize.py launches gpurun_out/r1_launches.csv "config 2"  > profiles/..._summary.txt
  python tools/summarize.py kernels  gpurun_out/r1_prof_c2.ncu-rep "config 2" > profiles/..._kernels.txt
  python tools/summarize.py traffic  gpurun_out/r1_prof_c2.ncu-rep           (per-kernel DRAM bytes, JSON)
"""

from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict


OURS = ("ring_interp_kernel", "strided_box_kernel", "box_copy_kernel", "restrict_reg_kernel", "gram_slide_kernel", "tile_interp_kernel", "tile3_interp_kernel", "tile3p_interp_kernel", "stage_slide_kernel", "window_kernel", "dense_apply_kernel",
        "tensor_apply_kernel", "finite_kernel", "csr_apply_kernel")
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "Kbyte/block": 1e3, "byte/block": 1.0}


def short(name: str) -> str:
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::|\(int\)|\(bool\)", "", name)
    name = name.split("(")[0] if "<" not in name.split("(")[0] else name[: name.index(">") + 1]
    return name.replace("void ", "").strip()


def launches(path: str, label: str) -> str:
    rows = [r for r in csv.reader(open(path)) if r]
    head = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[head]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg: "OrderedDict[str, list]" = OrderedDict()
    for r in rows[head + 1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        agg.setdefault(short(r[ki]), []).append(us)
    ours = {k: v for k, v in agg.items() if k.startswith(OURS)}
    tot = sum(sum(v) for v in ours.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none -> launch list ({label})",
           f"# cold-cache serialised launch times: compare shares, not absolutes; total of our kernels {tot:.1f} us"]
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:<55} launches {len(v):3d}  total {sum(v):9.1f} us  share {100 * sum(v) / tot:5.1f}%  "
                   f"mean {sum(v) / len(v):8.1f} us")
    return "\n".join(out)


def _raw(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    _val.units = units
    return h, [r for r in rows[2:] if r]


def _val(h, r, name):
    """Metric value in base units (us for durations, bytes for sizes)."""
    try:
        i = h.index(name)
        return float(r[i].replace(",", "")) * SCALE.get(_val.units[i], 1.0)
    except (ValueError, IndexError):
        return float("nan")


def kernels(rep: str, label: str) -> str:
    h, rows = _raw(rep)
    out = [f"# ncu --set full --clock-control none ({label})"]
    for r in rows:
        name = short(r[h.index("Kernel Name")])
        dur = _val(h, r, "gpu__time_duration.sum")
        rd = _val(h, r, "dram__bytes_read.sum")
        wr = _val(h, r, "dram__bytes_write.sum")
        out.append(name)
        out.append(f"   duration {dur:.1f} us, dram read {rd / 1e9:.3f} GB, write {wr / 1e9:.3f} GB, "
                   f"dram {(rd + wr) / dur / 1e3:.0f} GB/s ({_val(h, r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of peak), "
                   f"warps active {_val(h, r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%, "
                   f"regs {_val(h, r, 'launch__registers_per_thread'):.0f}, "
                   f"issue active {_val(h, r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%, "
                   f"smem/CTA {_val(h, r, 'launch__shared_mem_per_block_dynamic') / 1024:.1f} KB")
    return "\n".join(out)


def traffic(rep: str) -> str:
    h, rows = _raw(rep)
    res = OrderedDict()
    for r in rows:
        res[short(r[h.index("Kernel Name")])] = _val(h, r, "dram__bytes_read.sum") + _val(h, r, "dram__bytes_write.sum")
    return json.dumps(res, indent=1)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        print(launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""))
    elif cmd == "kernels":
        print(kernels(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""))
    elif cmd == "traffic":
        print(traffic(sys.argv[2]))
