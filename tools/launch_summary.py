"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) per kernel: count, median time,
share of the summed kernel time, median DRAM read/write per launch. Usage: launch_summary.py file.csv"""
import collections
import csv
import statistics
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    seq = [(k.split("(")[0].replace("void ", ""), m) for (i, k), m in d.items()]
    agg = collections.defaultdict(list)
    for n, m in seq:
        agg[n].append(m)
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, m in seq)
    print(f"{len(seq)} launches, summed kernel time {tot / 1e3:.1f} us")
    print("| kernel | launches | median us | share | DRAM read MB | DRAM write MB |")
    print("|---|---|---|---|---|---|")
    for n, v in sorted(agg.items(), key=lambda x: -sum(m.get("gpu__time_duration.sum", 0) for m in x[1])):
        t = [m.get("gpu__time_duration.sum", 0) for m in v]
        print(f"| {n} | {len(v)} | {statistics.median(t) / 1e3:.1f} | {sum(t) / tot:.3f} | "
              f"{statistics.median([m.get('dram__bytes_read.sum', 0) for m in v]) / 1e6:.1f} | "
              f"{statistics.median([m.get('dram__bytes_write.sum', 0) for m in v]) / 1e6:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
