# time the c5 .mns read/write (tools/stream_time.py) with each variant library under tools/var
for lib in tools/var/*.so; do
  echo "$lib $(MNS_B200_LIB=$PWD/$lib timeout 300 python tools/stream_time.py 2>&1 | tail -1)"
done
