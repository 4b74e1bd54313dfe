for r in 1 2; do for L in new m16 m24; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python bench.py --op residual --config 8 --steps 3 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('res c8 $L', round(d['ms_per_step'],3), 'ms')"
done; done
