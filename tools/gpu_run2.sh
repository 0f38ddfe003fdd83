cd $GRAFT_REPO_ROOT
./tools/umma_probe > gpurun_out/r2_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/r2_probe.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r2_ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cbm_kernel -s 1 -c 1 -o gpurun_out/r2_cfg4_cbm python tools/ncu_workload.py cfg4_b256 2 > gpurun_out/r2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu.log
