cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dense_gpu.py tests/test_hub_gpu.py -m gpu -q > gpurun_out/r42_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r42_pytest.log
timeout 1500 python bench.py > gpurun_out/r42_bench.json 2> gpurun_out/r42_bench.err; echo "bench rc=$?" >> gpurun_out/r42_bench.err
