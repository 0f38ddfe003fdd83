cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_hub_gpu.py -m gpu -q -x > gpurun_out/r29_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r29_pytest.log
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":16}}' '{"_env":{"CBM_B200_DENSE_DBG":31}}' > gpurun_out/r29_cfg3.jsonl 2> gpurun_out/r29_cfg3.err
unset CBM_B200_DENSE_DBG
REPS=12 timeout 1500 python tools/time_workload.py cfg4_b256 '{}' > gpurun_out/r29_cfg4.jsonl 2> gpurun_out/r29_cfg4.err
CBM_B200_DENSE_TRACE=gpurun_out/r29_dense_trace.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 '{}' > /dev/null 2> gpurun_out/r29_trace.err
