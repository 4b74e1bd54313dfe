for c in 3 7; do for r in 1 2; do for L in new t12 t24; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c $L', round(d['roofline']['kernel_ms']['k_fused2d']*1000,1), 'us')"
done; done; done
