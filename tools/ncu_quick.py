"""Print the key metrics + stall breakdown + pipe utilisation of one ncu report (no GPU):
  python tools/ncu_quick.py gpurun_out/x.ncu-rep"""
import csv
import subprocess
import sys

txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(txt.splitlines()))
h, u = rr[0], rr[1]
for v in rr[2:]:
    print("==", v[h.index("Kernel Name")][:60])
    for k in ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread", "launch__occupancy_limit_registers"]:
        if k in h:
            print(f"  {k} = {v[h.index(k)]} {u[h.index(k)]}")
    for i, x in enumerate(h):
        if x.startswith("sm__pipe_") and x.endswith("cycles_active.avg.pct_of_peak_sustained_active"):
            try:
                if float(v[i]) > 1:
                    print(f"  {x} = {v[i]}")
            except ValueError:
                pass
        if x.startswith("sm__inst_executed_pipe_") and x.endswith(".avg.pct_of_peak_sustained_active"):
            try:
                if float(v[i]) > 1:
                    print(f"  {x} = {v[i]}")
            except ValueError:
                pass
    st = {}
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            try:
                st[x] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    T = sum(st.values()) or 1.0
    for k, x in sorted(st.items(), key=lambda a: -a[1])[:12]:
        print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {x / T * 100:5.1f} %")
