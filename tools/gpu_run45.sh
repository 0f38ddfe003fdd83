cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_gcn_gpu.py -m gpu -q -x > gpurun_out/r45_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r45_pytest.log
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_L2_PERSIST":1}}' '{"_env":{"CBM_B200_L2_PERSIST":0}}' '{"_env":{"CBM_B200_L2_PERSIST":1,"CBM_B200_DENSE_DBG":32}}' '{"_env":{"CBM_B200_L2_PERSIST":0,"CBM_B200_DENSE_DBG":32}}' > gpurun_out/r45_cfg3.jsonl 2> gpurun_out/r45_cfg3.err
unset CBM_B200_DENSE_DBG
CBM_B200_L2_PERSIST=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:'cbm_kernel' -s 2 -c 1 python tools/ncu_workload.py cfg3 3 > gpurun_out/r45_ncu_cfg3_persist.txt 2>&1
