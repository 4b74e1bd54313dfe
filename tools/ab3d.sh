# per-phase A/B of the fused 3D kernel (dbg bits skip phases; results invalid, timing only)
for c in ${CONFIGS:-5 4}; do for o in 0 1 2 4 8 16 32 63; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --opt dbg=$o 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c$c dbg=$o', round(d['roofline']['kernel_ms']['k_fused3d'],2))"; done; done
