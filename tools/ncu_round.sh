# ncu evidence for the round: launch list of the default bench command + one --set full capture of
# the dominant kernel per config.  usage: TAG=r01 [CONFIGS="2 3 4 5"] bash tools/ncu_round.sh
TAG=${TAG:-r01}; mkdir -p gpurun_out
python bench.py > gpurun_out/plain_default.json 2> gpurun_out/plain_default.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches_default.csv \
    python bench.py > gpurun_out/ncu_launch.log 2>&1; echo launches_rc=$?
for c in ${CONFIGS:-2 3 4 5}; do
  if [ $c -ge 4 ]; then K=k_fused3d; else K=k_fused2d; fi
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c$c.json 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/${TAG}_c${c}_$K \
      python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c$c.log 2>&1; echo c$c full_rc=$?
done
