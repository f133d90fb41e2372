"""Dynamic SASS opcode histogram of one kernel launch in an ncu report (source page, SASS view)."""
import collections, csv, subprocess, sys

rep, kname = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
norm = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name",
                      f"regex:{kname}", "--launch-skip", skip, "--launch-count", "1"], capture_output=True,
                     text=True).stdout
hdr, cnt, tot = None, collections.Counter(), 0
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = r
        si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ii:
        continue
    try:
        n = int(r[ii] or 0)
    except ValueError:
        continue
    op = r[si].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    cnt[o.split(".")[0]] += n
    tot += n
print("total", tot, "per-unit", tot / norm)
for o, n in cnt.most_common(32):
    print(f"{o:10s} {n / norm:9.2f}  {n / tot * 100:5.1f}%")
