"""Hot SASS instructions of a kernel in an ncu report (--page source): top-N by stall samples, with executed
counts, and totals per opcode class. Reading aid for latency-bound kernels."""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first line: kernel name row; second: header
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
data = []
for r in rows[1:]:
    if len(r) <= iex or not r[ia].startswith("0x"):
        continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)))
base = data[0][0]
tot_s = sum(d[2] for d in data)
tot_e = sum(d[3] for d in data)
print(f"instructions {len(data)}, samples {tot_s}, warp instructions executed {tot_e}")
byop = collections.Counter()
byop_e = collections.Counter()
for a, s, n, e in data:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    op = op.split(".")[0]
    byop[op] += n
    byop_e[op] += e
print("by opcode (samples %, executed %):")
for op, n in byop.most_common(18):
    print(f"  {op:10s} {100*n/tot_s:5.1f}%  {100*byop_e[op]/tot_e:5.1f}%")
print("hottest instructions:")
for a, s, n, e in sorted(data, key=lambda d: -d[2])[:topn]:
    print(f"  +{a-base:05x} {100*n/tot_s:5.2f}%  exec {e:9d}  {s[:90]}")
