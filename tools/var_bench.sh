# time bench.py's c5 step with each variant library under tools/var (debug builds via MNS_B200_LIB)
for lib in tools/var/*.so; do
  MNS_B200_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-small --no-search > /tmp/vb.txt 2>&1
  echo "$lib $(python -c "import json,sys; d=json.loads(open('/tmp/vb.txt').read().strip().splitlines()[-1]); c=d['components']; print(round(d['ms_per_step'],4), round(c['encode_ms'],4), [round(x,4) for x in c['pass_ms_each']])" 2>&1 | tail -1)"
done
