# A/B of the 3D residual-only occupancy (variants/libiga_r*.so) against the package build
for c in 4 5; do for r in 1 2; do for L in new r6 r8; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --op residual --config $c --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('res c$c $L', round(d['ms_per_step'],3), 'ms')"
done; done; done
