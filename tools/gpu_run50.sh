cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel" -s 1 -c 1 -o gpurun_out/r50_cfg3_dense_full python tools/ncu_workload.py cfg3 3 > gpurun_out/r50_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cbm_kernel" -s 1 -c 1 -o gpurun_out/r50_cfg3_cold_full python tools/ncu_workload.py cfg3 3 > gpurun_out/r50_ncu2.log 2>&1
