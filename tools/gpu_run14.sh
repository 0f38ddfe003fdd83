cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/r14_dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r14_dense_tests.log
NOCHECK=1 REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":2}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":15}}' > gpurun_out/r14_cfg3.jsonl 2> gpurun_out/r14_cfg3.err
NOCHECK=1 REPS=3 CBM_B200_DENSE_TRACE=gpurun_out/r14_trace.txt timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' > /dev/null 2>&1
