"""Summarise an `ncu --set full` report for profiles/: per kernel the headline details (duration, DRAM
throughput, L2 hit rate, occupancy, ...) and the DRAM traffic per launch (dram__bytes_read.sum +
dram__bytes_write.sum), which bench.py reports as roofline.traffic.

  python tools/ncu_details.py gpurun_out/prof_cfg4.ncu-rep cfg4 profiles/r01_cfg4_ncu_full_details.json \
      profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

KEEP = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "L2 Hit Rate",
        "Issued Warp Per Scheduler", "No Eligible", "Block Size", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]
ROLE = {"k_local": "local", "k_local_panel": "local", "k_local_warp": "local", "k_local_inv": "local",
        "k_local_mrhs": "local", "k_local_mrhs_w": "local", "k_local_mrhs_r": "local", "k_local_mrhs_t": "local",
        "k_spmv3": "spmv", "k_spmv_ring": "spmv", "k_spmv_dd": "spmv", "k_spmv_cls": "spmv", "k_spmv_cls_t": "spmv"}


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True, check=True).stdout


def main(rep, cfg, details_out, traffic_out):
    det = {}
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(int)", "").strip()
        if r[mi] in KEEP:
            det.setdefault(name, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h = raw[0]
    traffic = {}
    for r in raw[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        base = name.split("<")[0]
        rd = float(d["dram__bytes_read.sum"].replace(",", ""))
        wr = float(d["dram__bytes_write.sum"].replace(",", ""))
        # raw units: ncu prints bytes scaled (Gbyte/Mbyte) in the header row 1
        units = dict(zip(h, raw[1]))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(units["dram__bytes_read.sum"], 1)
        wr *= scale.get(units["dram__bytes_write.sum"], 1)
        det.setdefault(name, {})["dram_bytes_per_launch"] = rd + wr
        if base in ROLE:
            traffic[ROLE[base]] = rd + wr
    json.dump(det, open(details_out, "w"), indent=1)
    try:
        allt = json.load(open(traffic_out))
    except Exception:
        allt = {}
    allt[cfg] = traffic
    json.dump(allt, open(traffic_out, "w"), indent=1)
    print(json.dumps(det, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
