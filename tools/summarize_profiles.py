"""Write profiles/<round>/ summaries from gpurun_out/ ncu artefacts (run here, no GPU):
  python tools/summarize_profiles.py r01 launches_r01e.csv k3_r01e.ncu-rep scan_r01e.ncu-rep
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, launches, k3rep = sys.argv[1:4]
scanrep = sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "-" else None
k3name = sys.argv[5] if len(sys.argv) > 5 else "k_exh_tiled"
out = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out, exist_ok=True)
src = os.path.join(ROOT, "gpurun_out")

rows = [r for r in csv.reader(open(os.path.join(src, launches))) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows:
    n = r[ki].split("(")[0]
    tot[n] += float(r[vi].replace(",", "")) / 1e6
    cnt[n] += 1
S = sum(tot.values())
lines = [f"# ncu launch list ({launches}): ncu --metrics gpu__time_duration.sum --clock-control none",
         "#   python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scaled [--no-next]",
         "# (3 device-resident + 3 e2e steps).  Per-launch times are cold-cache and serialised:",
         "# compare SHARES, not absolutes.",
         f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    lines.append(f"{k[:60]:60s} {cnt[k]:8d} {v:10.3f} {v / S * 100:6.1f}%")
lines.append(f"{'TOTAL':60s} {len(rows):8d} {S:10.3f}")
open(os.path.join(out, "launches_summary.txt"), "w").write("\n".join(lines) + "\n")

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers"]


def summary(rep, title):
    txt = subprocess.run(["ncu", "-i", os.path.join(src, rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(txt.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]
    res = [f"# {title} ({rep}, ncu --set full --clock-control none)"]
    vals = {}
    for k in KEYS:
        if k in h:
            res.append(f"{k} = {v[h.index(k)]} {u[h.index(k)]}")
            vals[k] = (v[h.index(k)], u[h.index(k)])
    st = {}
    for i, x in enumerate(h):
        if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued"):
            try:
                st[x] = float(v[i].replace(",", ""))
            except ValueError:
                pass
    T = sum(st.values()) or 1.0
    res.append("# warp-stall sampling (share of samples)")
    for k, x in sorted(st.items(), key=lambda a: -a[1])[:10]:
        res.append(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {x / T * 100:5.1f} %")
    return res, vals


k3, vals = summary(k3rep, f"{k3name}, exhaustive k=3, paper shape 1775 x 320, seed 1")
open(os.path.join(out, "k3_ncu_summary.txt"), "w").write("\n".join(k3) + "\n")
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
b = sum(float(vals[k][0].replace(",", "")) * unit.get(vals[k][1], 1)
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in vals)
l2 = float(vals["lts__t_sectors.sum"][0].replace(",", "")) * 32 if "lts__t_sectors.sum" in vals else None
l2pct = float(vals["lts__throughput.avg.pct_of_peak_sustained_elapsed"][0]) \
    if "lts__throughput.avg.pct_of_peak_sustained_elapsed" in vals else None
json.dump({"kernel": f"{k3name} k=3 paper shape", "bytes_per_launch": b,
           "l2_bytes_per_launch": l2, "l2_throughput_pct_of_peak": l2pct,
           "source": f"profiles/{rnd}/k3_ncu_summary.txt (dram__bytes_read.sum + dram__bytes_write.sum; "
                     "lts__t_sectors.sum x 32 B; lts__throughput)"},
          open(os.path.join(ROOT, "profiles", "k3_dram_bytes.json"), "w"), indent=1)
sc = []
if scanrep:
    sc, _ = summary(scanrep, "k_greedy_scan, scaled greedy step (65,536 configs x 4,096 envs, 1 GiB fp32 stream)")
    open(os.path.join(out, "scan_ncu_summary.txt"), "w").write("\n".join(sc) + "\n")
print("\n".join(lines[-6:]))
print("\n".join(k3[:8]))
print("\n".join(sc[:12]))
