"""Per-region instruction / stall-sample breakdown of one kernel from an ncu report (source page,
CUDA + SASS view): python tools/ncu_lines.py REPORT FILE.cu [norm] [top]."""
import csv
import re
import subprocess
import sys

rep, fname = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, res = None, []
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            res.append((int(r[7]), int(r[4]), cur, int(r[0])))
        except ValueError:
            pass
tot = sum(x[0] for x in res)
samp = sum(x[1] for x in res) or 1
src = open(fname).read().split("\n")
marks = []
for i, line in enumerate(src, 1):
    if re.match(r"^(__device__|__global__)", line) or re.search(r"auto (\w+) = \[", line) or \
            re.search(r"^\s+// (----|level|the 16)", line):
        marks.append((i, line.strip()[:70]))
base = fname.split("/")[-1]


def region(f, ln):
    if f != base:
        return "other:" + f
    name = "?"
    for i, t in marks:
        if i <= ln:
            name = f"{i}:{t}"
    return name


agg = {}
for n, s, f, ln in res:
    k = region(f, ln)
    agg.setdefault(k, [0, 0])
    agg[k][0] += n
    agg[k][1] += s
print(f"total {tot} warp-instr, {tot / norm:.1f} per unit")
for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    print(f"{n / norm:8.1f}/unit {n / tot * 100:5.1f}%  smp {s / samp * 100:5.1f}%  {k}")
