# time the c5 encode (tools/prof_encode.py) with each variant library under tools/var
for rep in 1 2; do
for lib in tools/var/*.so; do
  echo "$lib $(MNS_B200_LIB=$PWD/$lib timeout 300 python tools/prof_encode.py 2>&1 | tail -1)"
done
done
