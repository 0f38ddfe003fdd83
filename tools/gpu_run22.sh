cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hub_gpu.py -m gpu -q -x > gpurun_out/r22_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r22_pytest.log
REPS=12 timeout 1500 python tools/time_workload.py cfg4_b256 '{"hub":-1}' '{"hub":0}' > gpurun_out/r22_cfg4_hub.jsonl 2> gpurun_out/r22_cfg4_hub.err
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{"hub":-1}' '{"hub":0}' > gpurun_out/r22_cfg2_hub.jsonl 2> gpurun_out/r22_cfg2_hub.err
