# A/B of fused 3D occupancy variants (variants/libiga_*.so) against the package build
for r in 1 2; do
for L in new nh4 nh5; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 $L', round(d['roofline']['kernel_ms']['k_fused3d'],3), 'ms')"
done
for L in new ch12; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --config 8 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c8 $L', round(d['roofline']['kernel_ms']['k_fused3d'],3), 'ms')"
done; done
