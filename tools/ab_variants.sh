# time each variants/libiga_*.so on the given configs: CONFIGS="5 4" bash tools/ab_variants.sh
for v in variants/libiga_*.so; do for c in ${CONFIGS:-5 4}; do
  IGA_LIB=$PWD/$v python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); k=[x for x in d['roofline']['kernel_ms'] if x.startswith('k_fused')][0]; print('$v', 'c$c', round(d['roofline']['kernel_ms'][k],3), round(d['roofline']['step_frac'],4))"
done; done
