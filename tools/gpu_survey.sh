set -x
python -c "
import json, paper_1305_4452_b200 as iga
r = iga.microbench(0)
r2 = iga.microbench(0, 3, 1<<30); r['red_warp_8GB'] = r2['red_f64_warp_contig_per_s']
print(json.dumps(r, indent=1))
" > gpurun_out/microbench.json 2>&1
cat gpurun_out/microbench.json
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "cfg $c rc=$?"; cat gpurun_out/bench_c$c.json | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['value'], d['roofline']['kernel_ms'], d['roofline']['step_frac'])"; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_contract -s 1 -c 1 -o gpurun_out/prof_c2_contract python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
