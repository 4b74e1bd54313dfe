# ncu evidence for the round-1 additions: k_fused3d on config 8 (3D CH), the GMRES kernels on config 3
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT=$?; tail -6 gpurun_out/smoke.log
python bench.py --config 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c8.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fused3d -s 2 -c 1 -o gpurun_out/r01k_c8_k_fused3d \
    python bench.py --config 8 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c8.log 2>&1; echo c8_rc=$?
python tools/time_gmres.py --config 3 --reps 1 > gpurun_out/plain_gmres.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv_sw|k_ell_solve|k_multidot|k_multiaxpy" -s 40 -c 4 \
    -o gpurun_out/r01k_c3_k_gmres python tools/time_gmres.py --config 3 --reps 1 > gpurun_out/ncu_gmres.log 2>&1; echo gmres_rc=$?
