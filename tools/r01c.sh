TAG=r01c CONFIGS="2 3 5" bash tools/ncu_round.sh
for o in 0 1 2 3; do python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --opt dbg=$o 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 dbg=$o', round(d['ms_per_step'],2), d['roofline']['kernel_ms'])"; done
for o in 0 1 2 3; do python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --opt dbg=$o 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 dbg=$o', round(d['ms_per_step'],2), d['roofline']['kernel_ms'])"; done
