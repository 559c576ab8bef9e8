#!/usr/bin/env python
"""SASS instruction histogram of the hot per-iteration kernels in libdgas.so (CPU only: cuobjdump).

    python tools/sass_hist.py [--out profiles/r02_sass_hist.md]

For each hot kernel instantiation (the ones the BASELINE configs launch) it prints the instruction count,
the registers ptxas assigned, and the mnemonic classes that tell what the kernel is made of: FP64 math
(DFMA/DADD/DMUL), bulk-copy / mbarrier traffic (UBLKCP, SYNCS), plain global and shared loads/stores,
shuffles, barriers. Evidence for DESIGN.md §6 (TMA streaming, fp64 on the CUDA cores, no tensor-core
instructions on the iteration path)."""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1903_11357_b200", "libdgas.so")

# kernel-name regexes (demangled) -> where they run
HOT = [
    (r"k_spmv_ring<15>", "I1 SpMV, config 4 (byte ring)"),
    (r"k_spmv_cls_t<10>", "I1 SpMV, config 3 (class-sorted, de-duplicated A, FP64 tensor cores, default)"),
    (r"k_spmv_cls<10, 2>", "I1 SpMV, class-sorted on the CUDA cores (variant)"),
    (r"k_spmv_ring<28>", "I1 SpMV, config 5 p=6"),
    (r"k_local_mrhs_t<10>", "I5 local solves, config 3 (multi-RHS warp chains on the FP64 tensor cores, default)"),
    (r"k_local_mrhs_w<10, 2>", "I5 local solves, multi-RHS warp chains, K-slice lanes (variant)"),
    (r"k_local_mrhs_r<10>", "I5 local solves, multi-RHS, row lanes forward (variant)"),
    (r"k_local_mrhs<10>", "I5 local solves, multi-RHS, CTA-wide steps (variant)"),
    (r"k_local_panel<15, true, double, false>", "I5 local solves, config 4 (merged panels, narrow CTAs)"),
    (r"k_local_panel<10, false, double, true>", "I5 local solves, config 5 p = 3 (merged panels, wide CTAs, fused residual)"),
    (r"k_local_warp<10>", "I5 local solves, warp per subdomain"),
    (r"k_local_inv\(", "I5 local solves, explicit inverses (configs 1, 2, 5 p1)"),
    (r"k_local<28>", "I5 local solves, envelope kernel (p >= 5)"),
    (r"k_restrict_chunk<15, 6>", "I2+I3 update + restriction, config 4"),
    (r"k_restrict_chunk<10, 3>", "I2+I3 update + restriction, config 3"),
    (r"k_prolong<15, 6>", "I6 prolongation + r.z, config 4"),
    (r"k_prolong<10, 3>", "I6 prolongation + r.z, config 3"),
    (r"k_nd_fwd2|k_nd_bwd2|k_nd_fwd|k_nd_bwd", "I4 coarse solve, ND levels"),
    (r"k_coarse\(", "I4 coarse solve, dense inverse"),
    (r"k_pupdate", "I7 direction update (split)"),
    (r"k_lanczos", "I8 Lanczos"),
]
CLASSES = [
    ("fp64 math", r"^(DFMA|DADD|DMUL|DSETP|DMNMX)"),
    ("bulk copy (TMA)", r"^(UBLKCP|UBLKPF|UTMA)"),
    ("mbarrier", r"^SYNCS"),
    ("cp.async", r"^(LDGSTS|LDGDEPBAR|DEPBAR)"),
    ("global ld", r"^(LDG|LD\.)"),
    ("global st", r"^(STG|ST\.)"),
    ("atomics/red", r"^(ATOM|RED|ATOMG)"),
    ("shared ld", r"^LDS"),
    ("shared st", r"^STS"),
    ("shuffle", r"^SHFL"),
    ("barrier", r"^(BAR|WARPSYNC)"),
    ("tensor core", r"^(HMMA|DMMA|IMMA|UTC|TCGEN|QMMA|OMMA)"),
    ("branch", r"^(BRA|BRX|JMP|CALL|RET|EXIT|BSSY|BSYNC)"),
    ("int/addr", r"^(IMAD|IADD|LEA|ISETP|LOP|SHF|MOV|UMOV|UIADD|UIMAD|ULEA|USHF|ULOP|SEL|R2UR|S2R|S2UR|CS2R|PRMT|I2F|F2I|VIADD|UISETP|PLOP|ULDC|LDC|IABS|IMNMX|VIMNMX|USEL|POPC|FLO|BREV|SGXT|UPRMT|UFLO|UPOPC|R2P|P2R|VOTE|VOTEU|MATCH|REDUX|NOP|LDCU|UP2UR|UR2UP|ELECT|ENDCOLLECTIVE|ACQBULK|CCTL|MEMBAR|FENCE|ERRBAR|NANOSLEEP|YIELD|I2FP|F2FP|MUFU|FMUL|FFMA|FADD|FSETP|F2F|FSEL|I2I|FMNMX|FCHK|UF2FP|HADD2|HFMA2|UCLEA|UGETNEXTWORKID|BMOV|BPT|B2R|R2B|LEPC|WARPGROUP)"),
]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


def parse():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for ln in sass.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_.]+)?)", ln)
        if m and cur:
            funcs[cur].append(m.group(1))
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    regs, cur = {}, None
    for ln in res.splitlines():
        m = re.search(r"Function (\S+):", ln)
        if m:
            cur = m.group(1)
        m = re.search(r"REG:(\d+)", ln)
        if m and cur:
            regs[cur] = int(m.group(1))
    return funcs, regs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_sass_hist.md"))
    args = ap.parse_args()
    funcs, regs = parse()
    names = list(funcs)
    dem = dict(zip(names, demangle(names)))
    lines = ["# SASS instruction histogram of the hot kernels (`tools/sass_hist.py`, cuobjdump -sass libdgas.so)", "",
             "Static counts per kernel instantiation (sm_100a). `UBLKCP` = `cp.async.bulk` (TMA bulk copy), `SYNCS` = "
             "mbarrier arrive/try_wait, `LDGSTS` = `cp.async`, `DMMA` = `mma.sync.m8n8k4.f64`. The single-RHS kernels are "
             "fp64 GEMV-class work on the CUDA cores; the multi-RHS local solve (shared factors) is a dense "
             "contraction and runs on the FP64 tensor cores (DESIGN.md §6).", ""]
    hdr = ["kernel", "role", "instr", "regs"] + [c for c, _ in CLASSES[:-1]] + ["other top mnemonics"]
    lines.append("| " + " | ".join(hdr) + " |")
    lines.append("|" + "---|" * len(hdr))
    for pat, role in HOT:
        for mang in names:
            d = dem[mang]
            if not re.search(r"\b" + pat, d):
                continue
            ins = funcs[mang]
            base = [i.split(".")[0] for i in ins]
            counts = collections.OrderedDict((c, 0) for c, _ in CLASSES)
            other = collections.Counter()
            for full, b in zip(ins, base):
                for c, rx in CLASSES:
                    if re.match(rx, b) or re.match(rx, full):
                        counts[c] += 1
                        break
                else:
                    other[b] += 1
            short = re.sub(r"\(.*", "", d).replace("void ", "")
            row = [f"`{short}`", role, str(len(ins)), str(regs.get(mang, "?"))]
            row += [str(counts[c]) for c, _ in CLASSES[:-1]]
            row.append(", ".join(f"{k} {v}" for k, v in other.most_common(4)))
            lines.append("| " + " | ".join(row) + " |")
    open(args.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
