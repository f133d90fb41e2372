"""Issue-active %, duration and the top warp-stall reasons of the first kernel in an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
d = dict(zip(rows[0], rows[2]))
for k in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"):
    print(k, d.get(k))
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("_not_issued"):
        try:
            st.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", ""))))
        except ValueError:
            pass
tot = sum(x for _, x in st) or 1
for k, x in sorted(st, key=lambda t: -t[1])[:10]:
    print(f"  {k:24s} {x / tot * 100:5.1f}%")
