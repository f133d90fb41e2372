import csv, sys
from collections import defaultdict
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
d=defaultdict(list)
for r in rows[1:]:
    try: d[r[ki][:60]].append(float(r[vi].replace(",","")))
    except: pass
for k,v in sorted(d.items(), key=lambda x:-sum(x[1])): print(len(v), round(sum(v)/1e3,1), "us total", round(max(v)/1e3,1), "max", k)
