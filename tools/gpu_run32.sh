cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/umma_rate > gpurun_out/r32_umma_rate.txt 2>&1
timeout 900 python tools/probe_e2e_sweep.py cfg4_b256 default 4 > gpurun_out/r32_e2e.txt 2> gpurun_out/r32_e2e.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host" > gpurun_out/r32_pytest_host.log 2>&1; echo "rc=$?" >> gpurun_out/r32_pytest_host.log
