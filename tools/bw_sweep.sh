# L2-block width sweep of the 3D kernel: time (bench) and DRAM bytes (ncu, one launch) per bw.
#   BWS="2 4 7 12" [CONFIG=5] bash tools/bw_sweep.sh
mkdir -p gpurun_out/bw
for bw in ${BWS:-2 3 5 7 10 16}; do
  timeout 300 python bench.py --config ${CONFIG:-5} --steps 3 --warmup 3 --no-cpu-baseline --opt bw=$bw > gpurun_out/bw/bw$bw.json 2>/dev/null
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum --clock-control none -k regex:k_fused3d -s 3 -c 1 --csv \
      python bench.py --config ${CONFIG:-5} --steps 1 --warmup 3 --no-cpu-baseline --opt bw=$bw > gpurun_out/bw/ncu_bw$bw.csv 2>/dev/null
  python - <<PY
import json, csv
d = json.load(open("gpurun_out/bw/bw$bw.json"))
rows = [r for r in csv.reader(open("gpurun_out/bw/ncu_bw$bw.csv")) if len(r) > 10]
h = rows[0]; vals = {r[h.index("Metric Name")]: (r[h.index("Metric Value")], r[h.index("Metric Unit")]) for r in rows[1:]}
print("bw $bw", round(d["roofline"]["kernel_ms"]["k_fused3d"], 2), "ms", {k: v for k, v in vals.items()})
PY
done
