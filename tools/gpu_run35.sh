cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_hub_gpu.py -m gpu -q -x > gpurun_out/r36_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r36_pytest.log
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":16}}' > gpurun_out/r36_cfg3.jsonl 2> gpurun_out/r36_cfg3.err
unset CBM_B200_DENSE_DBG
CBM_B200_DENSE_TRACE=gpurun_out/r36_trace_full.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 '{}' > /dev/null 2> gpurun_out/r36_trace.err
python tools/trace_dense.py gpurun_out/r36_trace_full.txt > gpurun_out/r36_trace_full_summary.txt 2>&1
