bash tools/full_check.sh
TAG=r01j CONFIGS="2 3 4 5" bash tools/ncu_round.sh
for c in 2 3; do python bench.py --op basis3 --config $c --steps 10 --warmup 3 > gpurun_out/basis3_c$c.json 2>&1; done
for c in 2 3 4 5; do python bench.py --op residual --config $c --steps 10 --warmup 3 > gpurun_out/residual_c$c.json 2>&1; done
python tools/time_nsk.py > gpurun_out/nsk.json 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/reference.json 2>&1
