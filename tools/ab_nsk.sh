# A/B of the NSK fused kernel occupancy (variants/libiga_n*.so) against the package build
for r in 1 2; do for L in new q0; do
  if [ $L = new ]; then LIBV=""; else LIBV="IGA_LIB=$PWD/variants/libiga_$L.so"; fi
  env $LIBV python tools/time_nsk.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nsk $L', round(d['ms_per_step']*1000,1), 'us')"
done; done
