# A/B of the residual-only path: package build vs variants/libiga_base.so
for c in ${CONFIGS:-2}; do for r in 1 2; do for L in base new; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --op residual --config $c --steps 20 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('res c$c $L', round(d['ms_per_step']*1000,1), 'us')"
done; done; done
