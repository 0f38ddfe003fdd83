cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_hub_gpu.py -m gpu -q -x > gpurun_out/r43_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r43_pytest.log
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":256}}' '{"_env":{"CBM_B200_DENSE_DBG":16}}' '{"_env":{"CBM_B200_DENSE_DBG":272}}' > gpurun_out/r43_cfg3.jsonl 2> gpurun_out/r43_cfg3.err
