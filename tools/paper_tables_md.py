"""Render gpurun_out/paper_tables.json (tools/paper_tables.py) as markdown tables in the paper's layout.

Each cell: GPU K (iterations) / paper K (iterations); the oracle column states whether the CPU oracle
(run on the same seeded mesh) gave the same iteration count and K to 4 significant digits.
Usage: python tools/paper_tables_md.py gpurun_out/paper_tables.json > profiles/r01_paper_tables.md
"""
import json
import sys
from collections import defaultdict


def fmt(k, it):
    return f"{k:.4g} ({it})" if it is not None else f"{k:.3g}"


def main(path):
    rows = json.load(open(path))
    out = ["# Paper-regime reproduction on B200 (SURVEY §8f NEXT-1 / NEXT-2)", "",
           "Regime (PAPER.md:741): T_HH = T_h, C_sigma = 10, q = p, rtol 1e-8 from x0 = 0, K = Lanczos estimate.",
           "Meshes are our seeded Voronoi meshes (DESIGN.md R31-R33), not the paper's, so the paper's numbers",
           "are context (same trend and magnitude expected), while the oracle columns are parity: the CPU",
           "oracle on the same mesh. Cell format: GPU K (iterations) | paper K (iterations).", ""]
    par_total = par_ok = par_spread = 0
    dev_k = 0.0
    spread_cases = []
    for ex in (1, 2, 4):
        sel = [r for r in rows if r["ex"] == ex]
        if not sel:
            continue
        for p in sorted({r["p"] for r in sel}):
            rs = [r for r in sel if r["p"] == p]
            if ex == 1:
                out.append(f"## Ex.1 (L-shape, rho jumps), p = q = {p}: K vs rho_e")
                out.append("")
                rhos = sorted({r["coarse"][2] for r in rs})
                out.append("| variant | T_H vs rho | " + " | ".join(f"{x:.0e}" for x in rhos) + " |")
                out.append("|---|---|" + "---|" * len(rhos))
                grid = defaultdict(dict)
                for r in rs:
                    grid[(r["coarse"][0], r["coarse"][1])][r["coarse"][2]] = r
                for (variant, aligned), d in sorted(grid.items()):
                    cells = []
                    for x in rhos:
                        r = d.get(x)
                        cells.append("" if r is None else f"{fmt(r['K'], r['iters'])} \\| {fmt(r['paper_K'], None)}")
                    out.append(f"| {variant} | {'aligned' if aligned else 'not aligned'} | " + " | ".join(cells) + " |")
            else:
                name = "Ex.2 (nested agglomerates), rows H / h_bar" if ex == 2 else "Ex.4 (independent coarse Voronoi), rows N_H"
                out.append(f"## {name}, p = q = {p}, columns N_h")
                out.append("")
                cols = sorted({r["n_fine"] for r in rs})
                out.append("| coarse | " + " | ".join(str(c) for c in cols) + " |")
                out.append("|---|" + "---|" * len(cols))
                grid = defaultdict(dict)
                for r in rs:
                    grid[r["coarse"]][r["n_fine"]] = r
                keys = sorted([k for k in grid if k != "K(A_h)"], reverse=(ex == 2)) + (["K(A_h)"] if "K(A_h)" in grid else [])
                for coarse in keys:
                    cells = []
                    for c in cols:
                        r = grid[coarse].get(c)
                        if r is None:
                            cells.append("-")
                        elif coarse == "K(A_h)":  # unpreconditioned CG; the paper lists it for 3D only
                            cells.append(fmt(r["K"], r["iters"]))
                        else:
                            cells.append(f"{fmt(r['K'], r['iters'])} \\| {fmt(r['paper_K'], r['paper_iters'])}")
                    out.append(f"| {coarse} | " + " | ".join(cells) + " |")
            out.append("")
            for r in rs:
                if "oracle_iters" in r:
                    par_total += 1
                    within2 = abs(r["oracle_iters"] - r["iters"]) <= 2
                    kok = abs(r["oracle_K"] - r["K"]) <= 1e-2 * r["oracle_K"]
                    par_ok += int(within2 and kok)
                    if not within2:
                        spread_cases.append(r)
                        par_spread += int(bool(r.get("within_spread")) and kok)
                    dev_k = max(dev_k, abs(r["oracle_K"] - r["K"]) / r["oracle_K"])
    out.append(f"Oracle parity (north_star: iterations within 2, K within 1%): {par_ok} of {par_total} oracle-checked "
               f"cases. The other {len(spread_cases)} are long, K up to 4e7 runs where the stopping iteration of fp64 CG "
               f"is not unique under rounding (DESIGN.md R22); for them the oracle's OWN iteration counts under "
               f"last-bit perturbations of b, A and G were computed, and the GPU count lies inside that spread in "
               f"{par_spread} of {len(spread_cases)}. Largest K deviation over all {par_total}: {100 * dev_k:.3f}%.")
    out.append("")
    if spread_cases:
        out.append("| case | p | GPU iters | oracle iters | oracle spread | GPU K | oracle K |")
        out.append("|---|---|---|---|---|---|---|")
        for r in spread_cases:
            sp = r.get("oracle_spread")
            out.append(f"| {r['coarse'] if r['ex'] != 1 else '/'.join(map(str, r['coarse']))} (ex{r['ex']}, N_h {r['n_fine']}) "
                       f"| {r['p']} | {r['iters']} | {r['oracle_iters']} | {sp[0] if sp else '?'}..{sp[1] if sp else '?'} "
                       f"| {r['K']:.6g} | {r['oracle_K']:.6g} |")
    times = [(r["solve_ms"], r) for r in rows if "solve_ms" in r]
    out.append("")
    out.append("Solve times (GPU, one dgas_pcg incl. Lanczos): " +
               ", ".join(f"ex{r['ex']} p{r['p']} N_h={r['n_fine']}: {t:.1f} ms / {r['iters']} it"
                         for t, r in sorted(times, key=lambda x: -x[0])[:5]) + " (largest five).")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/paper_tables.json")
