python -c "
import json, paper_1305_4452_b200 as iga
r = iga.microbench(0)
for big in (1<<30,):
    for k in (3, 8, 9, 10):
        r[iga.MICROBENCH[k]+'_8GB'] = iga.microbench(0, k, big)[iga.MICROBENCH[k]]
print(json.dumps(r, indent=1))
" > gpurun_out/microbench2.json 2>&1; cat gpurun_out/microbench2.json
