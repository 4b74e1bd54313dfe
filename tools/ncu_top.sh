# usage: CFG=3 KREGEX=k_fused2d [N=32] [EXTRA="--opt dbg=3"] bash tools/ncu_top.sh
CFG=${CFG:-2}; K=${KREGEX:-k_fused2d}; OUT=${OUT:-prof_c${CFG}_${K}}
NARG=""; if [ -n "$N" ]; then NARG="--n $N"; fi
python bench.py --config $CFG $NARG $EXTRA --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/$OUT python bench.py --config $CFG $NARG $EXTRA --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu_rc=$?
