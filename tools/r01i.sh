bash tools/full_check.sh
TAG=r01i CONFIGS="2 3 4 5" bash tools/ncu_round.sh
for c in 2 3; do python bench.py --op basis3 --config $c --steps 10 --warmup 3 > gpurun_out/basis3_c$c.json 2>&1; done
