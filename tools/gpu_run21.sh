cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hub_gpu.py tests/test_dense_gpu.py -m gpu -q -x > gpurun_out/r21_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r21_pytest.log
REPS=12 timeout 1500 python tools/time_workload.py cfg4_b256 '{"hub":0}' '{"hub":-1}' '{"hub":-1,"_env":{"CBM_B200_BAND_COLS":24576}}' > gpurun_out/r21_cfg4_hub.jsonl 2> gpurun_out/r21_cfg4_hub.err
unset CBM_B200_BAND_COLS
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{"hub":0}' '{"hub":-1}' > gpurun_out/r21_cfg2_hub.jsonl 2> gpurun_out/r21_cfg2_hub.err
timeout 120 ./tools/ubench_gather4 > gpurun_out/r21_ubench_gather4.txt 2>&1; echo "rc=$?" >> gpurun_out/r21_ubench_gather4.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum -k regex:'cbm_kernel|dense_kernel|hub_reduce' -s 3 -c 3 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r21_ncu_cfg4_hub.txt 2>&1
