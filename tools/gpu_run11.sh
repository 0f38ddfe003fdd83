cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/r11_dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r11_dense_tests.log
NOCHECK=1 REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":1}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":2}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":7}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":0}}' > gpurun_out/r11_cfg3.jsonl 2> gpurun_out/r11_cfg3.err
timeout 600 python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r11_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_kernel" -s 1 -c 1 -o gpurun_out/r11_cfg3_dense python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r11_ncu.log 2>&1
