for lib in tools/var/*.so; do echo "$lib"; MNS_B200_LIB=$PWD/$lib timeout 300 python tools/f64_time.py 2>&1 | tail -4; MNS_B200_LIB=$PWD/$lib python tools/c2iso_prof.py; done
