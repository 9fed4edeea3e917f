"""Brief per-kernel ncu summary: stalls, instruction mix, occupancy.  python tools/ncu_brief.py rep.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d["Kernel Name"][:90])
    ks = [k for k in hdr if "warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")]
    st = sorted(((float(d[k].replace(",", "")) if d[k] else 0, k) for k in ks), reverse=True)[:7]
    print("   stalls/issue: " + ", ".join(f"{k.split('stalled_')[1].replace('_per_issue_active.ratio','')} {v:.2f}" for v, k in st))
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "dram__bytes_read.sum",
              "dram__bytes_write.sum", "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]:
        print(f"   {k} {d.get(k)}")
