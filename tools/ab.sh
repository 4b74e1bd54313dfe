# A/B timing of variant libraries (tools/variant.py) on the GPU box; optional parity subset.
#   VARS="base v1" CONFIGS="5 4" [PARITY="5-5 or 4-5"] [STEPS=3] bash tools/ab.sh
mkdir -p gpurun_out/ab
for v in $VARS; do
  for c in ${CONFIGS:-5}; do
    IGA_LIB=$PWD/scratch/libiga_$v.so timeout 300 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline $EXTRA > gpurun_out/ab/${v}_c$c.json 2>gpurun_out/ab/${v}_c$c.err
    python -c "import sys,json; d=json.load(open('gpurun_out/ab/${v}_c$c.json')); print('$v c$c', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['roofline']['kernel_ms'].items()}, 'frac %.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/ab/${v}_c$c.err
  done
  if [ -n "$PARITY" ]; then IGA_LIB=$PWD/scratch/libiga_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$PARITY" 2>&1 | tail -2; fi
done
