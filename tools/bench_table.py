"""Markdown table of bench.py JSON lines (gpurun_out/bench_*.log) for profiles/rNN_summary.md."""
import glob
import json
import os
import sys


def last_json(path):
    for line in reversed(open(path).read().splitlines()):
        line = line.strip()
        if line.startswith("{"):
            try:
                return json.loads(line)
            except Exception:
                return None
    return None


def main(d="gpurun_out"):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "bench_*.log"))):
        j = last_json(f)
        if not j or "kernels" not in j:
            continue
        rows.append((os.path.basename(f)[6:-4], j))
    print("| run | N | PCG it/s | e2e it/s | iters | Lanczos K | SpMV us | local us | coarse us | apply us | "
          "local kernel | roofline.frac (kernel) | t_env/t_meas |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name, j in rows:
        k, run = j["kernels"], j.get("run", {})
        ar = j.get("algorithmic_roofline_per_iter", {})
        print(f"| {name} | {j['config']['N']:,} | {j['value']:,.0f} | {j['e2e']['value']:,.0f} | "
              f"{run.get('iters_per_solve', 0):.0f} | {run.get('lanczos_cond', 0):.6g} | {1e3 * k['spmv']['ms']:.1f} | "
              f"{1e3 * k['local']['ms']:.1f} | {1e3 * k['coarse']['ms']:.1f} | {1e3 * k['apply_total']['ms']:.1f} | "
              f"{run.get('local_kernel')} | {j['roofline']['frac']:.3f} ({j['roofline']['kernel']}) | "
              f"{ar.get('t_env_over_t_measured', 0):.3f} |")


if __name__ == "__main__":
    main(*sys.argv[1:])
