#!/usr/bin/env python
"""bench.py — ASPCG throughput on B200 (BASELINE.json metric: PCG iters/s and the HBM GB/s of the
Schwarz-apply + SpMV kernels, fp64, 1 x B200, % of HBM peak).

A step = one full dgas_pcg solve (rtol 1e-8, x0 = 0) of the workload: every per-iteration row of
SURVEY.md §8(a) (SpMV, axpy/norm, restriction, coarse solve, local solves, prolongation, direction
update) plus the Lanczos estimate. value = PCG iterations per second over the K timed steps (inputs
already resident in HBM); e2e = the same metric through dgas_pcg_host (host b/x copied in and out
inside the timed region). Multi-GPU: independent replicas, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {  # name -> (BASELINE config index, p, q)
    "cfg1": (1, None, None), "cfg2": (2, None, None), "cfg3": (3, None, None), "cfg4": (4, None, None),
    **{f"cfg5_p{p}q{q}": (5, p, q) for p in range(1, 7) for q in sorted({1, p})},
}
METRIC = "PCG iters/s & Schwarz-apply+SpMV HBM GB/s (fp64, 1xB200), % of HBM peak"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _problem(name):
    import dgas_gen
    k, p, q = CONFIGS[name]
    return dgas_gen.config(k, p, q) if k == 5 else dgas_gen.config(k)


class Clocks:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    def __init__(self, idx):
        self.idx = idx
        self.proc = None
        self.path = os.path.join("/tmp", f"dgas_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines() if l.strip()]
            sm = sorted(float(r[0]) for r in rows)
            mx = max(float(r[1]) for r in rows)
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].strip() == "Active"})
            return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}
        except Exception:
            return None


def aggregate(ms, iters, world, device="cpu"):
    """Whole-job numbers over replicas: time = MAX over ranks, iterations = SUM over ranks."""
    if world <= 1:
        return ms, iters
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms, iters], dtype=torch.float64, device=device)
    mx = t.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def host_info():
    model = ""
    try:
        for l in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=20).stdout.splitlines():
            if l.startswith("Model name"):
                model = l.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "lscpu_model": model}


def l2_policy(P):
    """Deterministic from the problem (both arms print the same config): the operators of one PCG
    iteration (A and the local factors, >= ~12 n_p-blocks per cell) against the B200's 126 MB L2."""
    est = 12 * P.N * P.n_p * 8
    vec = 6 * P.N * 8  # x, b, r, z, p, q
    if est > 126e6:
        return (f"inputs larger than L2 (per-iteration working set > 126 MB: six N-vectors {vec / 1e6:.0f} MB plus "
                f"the operators; no flush needed)")
    return f"L2-resident (operators ~{est / 1e6:.1f} MB fit the 126 MB L2; L2 flushed before every timed solve)"


def problem_config(name, P):
    return {"workload": name, "N": P.N, "N0": P.N0, "p": P.p, "q": P.q, "n_cells": P.n_cells,
            "n_subdomains": P.n_sub, "n_coarse": P.n_coarse, "rtol": 1e-8, "maxit": 5000, "x0": "zero",
            "l2_policy": l2_policy(P)}


class OracleSample:
    """The oracle (oracle/, test infrastructure) as it stands, timed on a bounded sample of one PCG
    iteration of the workload: the full SpMV, the full restriction + coarse solve (A0 factored in
    full, untimed setup), the local solves + prolongation of `ns` spread subdomains scaled to all
    n_sub, and the iteration's vector ops (3 axpys, 2 dots). Threads: OpenMP over subdomains."""

    def __init__(self, name, P, ns):
        import numpy as np

        import dgas_gen
        import oracle
        self.oracle = oracle
        self.P = P
        self.sub = sorted(set(np.linspace(0, P.n_sub - 1, min(ns, P.n_sub)).astype(int).tolist()))
        t0 = time.time()
        self.o = oracle.Oracle(P)
        self.o.setup_schwarz(sample=self.sub)
        self.t_setup = time.time() - t0
        self.x = dgas_gen.normal(1, self.o.N)

    def iteration_seconds(self, threads, reps=2):
        import numpy as np
        self.oracle.set_threads(threads)
        o, x, sub = self.o, self.x, self.sub

        def best(f):
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
            return min(ts)
        t_spmv = best(lambda: o.spmv(x))
        t_coarse = best(lambda: o.apply_sampled(x, []))           # restriction + coarse solve
        t_cs = best(lambda: o.apply_sampled(x, sub))              # + local solves, prolongation (sample)
        v = x.copy()

        def vec():
            v[:] += 0.5 * x; v[:] -= 0.25 * x; float(v @ x); v[:] = x + 0.1 * v; float(v @ v)
        t_vec = best(vec)
        return t_spmv + t_coarse + max(0.0, t_cs - t_coarse) * self.P.n_sub / len(self.sub) + t_vec

    def sample_text(self, name):
        return (f"{name}: one oracle PCG iteration = SpMV over all {self.P.n_cells} cells + restriction and "
                f"{'band' if self.P.N0 > 8192 else 'dense'}-Cholesky coarse solve of all N0 = {self.P.N0} + "
                f"dense-Cholesky local solves and prolongation of {len(self.sub)}/{self.P.n_sub} spread "
                f"subdomains scaled to all + vector ops (setup {self.t_setup:.0f}s untimed)")


def cpu_baseline(name, P=None):
    """Reported baseline (never the target): all host cores (OpenMP) and one core."""
    P = _problem(name) if P is None else P
    nproc = os.cpu_count() or 1
    smp = OracleSample(name, P, ns=max(8, min(64, 2 * nproc)))
    t_all = smp.iteration_seconds(nproc)
    t_one = smp.iteration_seconds(1)
    return {"value": 1.0 / t_all, "unit": "PCG it/s", "cores": nproc, "kind": "oracle",
            "sample": smp.sample_text(name), "host": host_info(),
            "single_core": {"value": 1.0 / t_one, "unit": "PCG it/s", "cores": 1}}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands on the host cores (this tier's reference arm)."""
    if rank != 0:
        return
    name = args.config
    P = _problem(name)
    nproc = os.cpu_count() or 1
    smp = OracleSample(name, P, ns=max(8, min(64, 2 * nproc)))
    for _ in range(args.warmup):
        smp.iteration_seconds(nproc, reps=1)
    per = [smp.iteration_seconds(nproc, reps=1) for _ in range(max(1, args.steps))]
    v = 1.0 / (sum(per) / len(per))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "PCG it/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(per) / len(per),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": problem_config(name, P),
            "cpu_baseline": {"value": v, "unit": "PCG it/s", "cores": nproc, "kind": "oracle",
                             "sample": smp.sample_text(name), "host": host_info()},
            "e2e": {"value": v, "unit": "PCG it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))  # the largest BASELINE config
    ap.add_argument("--impl", default="dgas", choices=["dgas", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas of the single-GPU solve instead of the sharded solve")
    ap.add_argument("--local-f32", action="store_true",
                    help="NEXT-4 variant outside the fp64 contract: fp32-stored local factors (never the headline)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0)); world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch

    if args.local_f32:
        os.environ["DGAS_PANEL_F32"] = "1"
        os.environ["DGAS_LOCAL_INV"] = "0"
    from paper_1903_11357_b200 import dgas
    # DGAS_BENCH_DEVICE / DGAS_DIST_BACKEND: test hooks (several ranks on one GPU over gloo)
    local = int(os.environ.get("DGAS_BENCH_DEVICE", local))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(os.environ.get("DGAS_DIST_BACKEND", "nccl"))
    P = _problem(args.config)
    t0 = time.time()
    S = dgas.Solver(P)
    torch.cuda.synchronize()
    t_setup = time.time() - t0
    info = S.info
    b = S.rhs(P.f_kind)
    x = torch.zeros_like(b)
    # N > 1: the subdomain-sharded solve over NCCL: one problem, total work fixed
    sharded = world > 1 and not args.replicas
    SS = dgas.ShardedSolver(S) if sharded else None

    def solve(bb, xx):
        if sharded:
            xs, it_, c_, st_ = SS.pcg(bb)
            xx.copy_(xs)
            return xx, it_, c_, st_
        return S.pcg(bb, xx)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        x.zero_(); solve(b, x)
    barrier()
    iters_total = 0
    iters_list = []
    conds = []
    # L2-resident workloads (config 1, 2, small config-5 pairs): flush L2 before every timed step by
    # writing a buffer twice its size (outside the step's events); larger workloads need no flush
    flush = None
    if l2_policy(P).startswith("L2-resident"):
        flush = torch.empty(2 * torch.cuda.get_device_properties(local).L2_cache_size // 4, dtype=torch.float32,
                            device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        barrier()
        for k in range(args.steps):
            x.zero_()
            if flush is not None:
                flush.fill_(float(k))
            ev[k][0].record()
            _, it, cond, st = solve(b, x)
            ev[k][1].record()
            iters_total += it
            iters_list.append(it)
            conds.append(cond)
        barrier()
    ms = sum(a.elapsed_time(c) for a, c in ev)
    ms, iters_all = aggregate(ms, iters_total, world, device="cuda")
    if sharded:
        iters_all = iters_total  # one shared solve: the ranks' iterations are the same iterations
    value = iters_all / (ms / 1e3)
    iters_per_solve = iters_total / args.steps

    # ---- e2e through the public C ABI with host buffers (pinned), copies inside the timed region
    bh = b.cpu().pin_memory()
    xh = torch.zeros(S.N, dtype=torch.float64).pin_memory()
    if sharded:  # host b in, solve, host x out (every rank holds b and receives x)
        def host_solve():
            bd = bh.to("cuda", non_blocking=True)
            xd, it_, _, _ = SS.pcg(bd)
            xh.copy_(xd)
            return it_
    else:
        def host_solve():
            return S.pcg_host(bh, xh)[0]
    host_solve()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    e2e_iters = 0
    for _ in range(args.steps):
        xh.zero_()
        e2e_iters += host_solve()
    e3.record()
    barrier()
    e2e_ms = e2.elapsed_time(e3)
    e2e_ms, _ = aggregate(e2e_ms, 0, world, device="cuda")
    e2e_value = e2e_iters * (1 if sharded else world) / (e2e_ms / 1e3)

    # ---- per-kernel timing (CUDA events on the launching stream) for the roofline
    peaks = _peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    stream = torch.cuda.current_stream()
    S.bench_kernels(0, 3); S.bench_kernels(2, 3)
    kt = {}
    for which, nm in ((0, "spmv"), (2, "apply_fused"), (1, "apply_total"), (3, "local"), (4, "coarse")):
        torch.cuda.synchronize()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        S.bench_kernels(which, args.kernel_reps)
        c.record(stream)
        torch.cuda.synchronize()
        kt[nm] = a.elapsed_time(c) / args.kernel_reps
    N, N0, npp = info["N"], info["N0"], info["n_p"]
    dinv_tri = info["n_cells"] * npp * (npp + 1) // 2 * 8
    alg = {
        "spmv": info["alg_bytes_spmv"],
        "apply_fused": info["bytes_local"] + info["bytes_coarse"] + 2 * N * 8 + 2 * N0 * 8,
        "apply_total": info["alg_bytes_apply"],
        "local": info["bytes_local"] + 2 * N * 8,
        "coarse": info["bytes_coarse"] + 2 * N0 * 8,
    }
    kern = {nm: {"ms": kt[nm], "alg_bytes": alg[nm], "GBps": alg[nm] / (kt[nm] * 1e-3) / 1e9,
                 "frac": alg[nm] / (kt[nm] * 1e-3) / 1e9 / hbm_peak} for nm in kt}
    # SURVEY §8(d) algorithmic minimum: A as its symmetric half (diagonal blocks' lower triangles, every
    # coupled pair once) next to the full block-CSR the kernel streams
    nnzb, nh = info["nnz_blocks"], info["n_cells"]
    a_sym = 8 * (nh * npp * (npp + 1) // 2 + (nnzb - nh) // 2 * npp * npp)
    kern["spmv"]["alg_bytes_sym_half"] = a_sym + 2 * N * 8
    kern["spmv"]["frac_sym_half"] = (a_sym + 2 * N * 8) / (kt["spmv"] * 1e-3) / 1e9 / hbm_peak
    # B_env of one PCG iteration: A symmetric half, local envelope factor once, coarse
    # factor (x refinement passes), Q twice, ~10 N vector entries; t_env = B_env / peak
    refine = info["coarse_refine"]
    b_env = (a_sym + info["bytes_U"] + dinv_tri + info["bytes_coarse"] * (1 + refine) + 2 * info["bytes_G"]
             + 10 * N * 8)
    t_iter_ms = ms / max(1, iters_total)
    dom = "local" if kt["local"] >= kt["spmv"] else "spmv"
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(args.config, {}).get(dom)
    except Exception:
        pass
    spmv_apply_gbs = (alg["spmv"] + alg["apply_total"]) / ((kt["spmv"] + kt["apply_total"]) * 1e-3) / 1e9
    # fp64 arithmetic of the dominant kernel against the FP64 peak from the unit counts (148 SMs x 64 FMA/clk x 2
    # flop at the SM clock: 37.2 TFLOP/s at 1965 MHz): every stored operator entry is one FMA per use
    # (SpMV: all stored blocks; local solves: factor + D triangles, forward and backward sweep)
    props = torch.cuda.get_device_properties(local)
    fp64_peak = props.multi_processor_count * 64 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    flops = {"spmv": 2.0 * nnzb * npp * npp, "local": 4.0 * (info["bytes_U"] + dinv_tri) / 8.0}
    alu = {"bound": "alu", "achieved": flops[dom] / (kt[dom] * 1e-3) / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
           "frac": flops[dom] / (kt[dom] * 1e-3) / 1e12 / fp64_peak,
           "note": ("fp64 FMA work of the same kernel against the FP64 peak derived from the unit counts (148 SMs x 64 "
                    "FMA/clk x 2 flop x SM clock; the guides give no separate FP64 tensor figure). "
                    + ("This kernel issues mma.sync.m8n8k4.f64 (FP64 tensor cores): a dense multi-right-hand-side "
                       "contraction; it is bound by the latency of its dependent chain, not by the math rate."
                       if dom == "local" and info["local_kernel"] == 5 else
                       "CUDA-core DFMA kernel (single right-hand side, GEMV-class)."))}

    line = {
        "metric": METRIC, "value": value, "unit": "PCG it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": problem_config(args.config, P),
        "run": {"iters_per_solve": iters_per_solve, "lanczos_cond": conds[-1] if conds else None,
                "parallelism": (f"sharded-subdomains-{world}x-nccl" if sharded else "replicas") if world > 1
                else "single-gpu", "setup_s": t_setup,
                "coarse_solver": ["dense-inverse", "band", "nested-dissection"][info["coarse_mode"]],
                "coarse_refine_steps": refine, "coarse_solve_relerr": info["coarse_solve_relerr"],
                "local_kernel": {1: "envelope", 2: "panel", 3: "explicit-inverse", 4: "warp-per-subdomain", 5: "multi-rhs-shared-factor"}.get(
                    info["local_kernel"]),
                "local_ctas_per_sm": info["local_ctas_per_sm"],
                "operator_bytes": info["bytes_A"] + info["bytes_U"] + info["bytes_coarse"] + info["bytes_G"],
                "l2_bytes": torch.cuda.get_device_properties(local).L2_cache_size},
        "algorithmic_roofline_per_iter": {
            "B_env_bytes": b_env, "t_env_ms": b_env / (hbm_peak * 1e9) * 1e3, "t_measured_ms": t_iter_ms,
            "t_env_over_t_measured": b_env / (hbm_peak * 1e9) * 1e3 / t_iter_ms,
            "note": "SURVEY §8(d) B_env (A symmetric half, envelope factor read once) at the measured HBM peak"},
        "dof_iters_per_s": value * N / max(world, 1) * world,
        "ms_per_apply": kt["apply_total"],
        "spmv_apply_hbm_gbs": spmv_apply_gbs,
        "spmv_apply_pct_of_hbm_peak": 100 * spmv_apply_gbs / hbm_peak,
        "roofline": {"bound": "hbm", "achieved": kern[dom]["GBps"], "peak": hbm_peak, "unit": "GB/s",
                     "frac": kern[dom]["frac"], "traffic": traffic, "kernel": dom,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6650 GB/s",
                     "alu": alu,
                     **({"note": (f"operators de-duplicated (exact, NEXT-4): A {info['dedup_A_bytes'] / 1e6:.1f} MB and "
                                  f"local factors {info['dedup_local_bytes'] / 1e6:.1f} MB stored, L2-resident; "
                                  f"'achieved' divides the SURVEY 8(d) algorithmic bytes (full envelope factor) by the "
                                  f"launch time (it can exceed the HBM peak: the shared operators are read from "
                                  f"L2, the kernel is instruction-bound), 'traffic' is what ncu measured from DRAM")}
                        if info.get("dedup_A_bytes") else {})},
        "kernels": kern,
        "e2e": {"value": e2e_value, "unit": "PCG it/s", "h2d_bytes_per_step": 2 * N * 8,
                "d2h_bytes_per_step": N * 8},
        # the last WHILE body of a solve also launches its remaining unrolled copies (immediate return)
        "gpu_launches": (int((info["launches_per_iter"] + 12) * sum(iters_list) + 16 * args.steps) if sharded else
                         int(info["launches_per_iter"] * sum(-(-it // info["unroll"]) * info["unroll"]
                                                             for it in iters_list)
                             + info["launches_per_solve"] * args.steps)),
        "clocks": clk.summary(),
    }
    if args.local_f32:
        line["variant"] = "NEXT-4: fp32-stored local factors, fp64 arithmetic (outside the fp64 contract; not the headline)"
        line["dtype"] = "f64 (local factors stored f32)"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb = cpu_baseline(args.config, P)
            cb.pop("seconds_per_iter", None)
            line["cpu_baseline"] = cb
        except Exception as e:  # the oracle is a reported baseline, never the target
            line["cpu_baseline"] = {"value": None, "unit": "PCG it/s", "cores": 1, "kind": "oracle",
                                    "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    S.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
