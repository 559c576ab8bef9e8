"""Print the headline metrics and the warp-stall breakdown of each kernel in an ncu report (reading aid)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
keys = sys.argv[2:] or ["Duration", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate", "Compute (SM) Throughput",
                        "Issued Warp Per Scheduler", "No Eligible", "Achieved Occupancy", "Theoretical Occupancy",
                        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
                        "Warp Cycles Per Issued Instruction", "Executed Ipc Active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
seen = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    k = (r[ii], r[ki].split("(")[0])
    if r[mi] in keys:
        seen.setdefault(k, []).append(f"{r[mi]}={r[vi]} {r[ui]}")
for k, v in seen.items():
    print(k[0], k[1])
    for x in v:
        print("   ", x)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh, units = rr[0], rr[1]
for row in rr[2:]:
    st = [(hh[i].replace("smsp__average_warp_latency_issue_stalled_", "").replace("smsp__pcsamp_warps_issue_stalled_", ""), row[i])
          for i in range(len(hh)) if hh[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hh[i].endswith("_not_issued")]
    tot = sum(float(v or 0) for _, v in st)
    top = sorted(st, key=lambda t: -float(t[1] or 0))[:8]
    print(row[hh.index("Kernel Name")][:40], "stall samples:", ", ".join(f"{n} {float(v)/max(tot,1):.0%}" for n, v in top))
