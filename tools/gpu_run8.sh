cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/r8_dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r8_dense_tests.log
NOCHECK=1 REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":1}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":2}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":7}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":0}}' > gpurun_out/r8_cfg3.jsonl 2> gpurun_out/r8_cfg3.err
