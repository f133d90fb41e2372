# for each variant library under tools/var: the lattice/strip/golden parity tests, then the c5 step timing
for lib in tools/var/*.so; do
  MNS_B200_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lattice or strip or golden" > /tmp/vt.txt 2>&1
  echo "$lib tests: $(tail -1 /tmp/vt.txt)"
done
bash tools/var_bench.sh
