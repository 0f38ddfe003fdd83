cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=12 timeout 1800 python tools/time_workload.py cfg4_b256 '{}' '{"split_threshold":256,"chunk":64}' '{}' '{"split_threshold":256,"chunk":64}' > gpurun_out/r47_cfg4_split.jsonl 2> gpurun_out/r47_cfg4_split.err
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_hub_gpu.py -m gpu -q -x > gpurun_out/r47_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r47_pytest.log
