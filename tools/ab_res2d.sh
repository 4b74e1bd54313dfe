# A/B: 2D residual-only occupancy variant (variants/libiga_r2.so) vs the package build
for c in 2 3 7; do for r in 1 2; do for L in new r2; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --op residual --config $c --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('res c$c $L', round(d['ms_per_step']*1000,1), 'us')"
done; done; done
