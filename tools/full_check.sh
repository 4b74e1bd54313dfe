# full GPU check: all parity tests, smoke, bench per config, launch list of the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT=$?
for c in ${CONFIGS:-1 2 3 4 5}; do timeout 600 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; python -c "import sys,json; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['config']['workload'], round(d['ms_per_step'],4), '%.3g'%d['value'], {k:round(v,4) for k,v in d['roofline']['kernel_ms'].items()}, 'frac %.4f'%d['roofline']['step_frac'])" || tail -3 gpurun_out/bench_c$c.err; done
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo BENCH_EXIT=$?; cat gpurun_out/bench_default.json
