cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dense_gpu.py tests/test_tile_gpu.py -m gpu -q -x > gpurun_out/r18_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r18_pytest.log
REPS=10 timeout 1200 python tools/time_workload.py cfg4_b256 '{"_env":{"CBM_B200_BAND_COLS":0}}' '{"_env":{"CBM_B200_BAND_COLS":49152}}' '{"_env":{"CBM_B200_BAND_COLS":24576}}' '{"_env":{"CBM_B200_BAND_COLS":98304}}' '{"_env":{"CBM_B200_BAND_COLS":49152},"chunk":128}' '{"_env":{"CBM_B200_BAND_COLS":49152},"chunk":256}' '{"_env":{"CBM_B200_BAND_COLS":49152},"max_segments":1}' > gpurun_out/r18_cfg4_band.jsonl 2> gpurun_out/r18_cfg4_band.err
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{"_env":{"CBM_B200_BAND_COLS":0}}' '{"_env":{"CBM_B200_BAND_COLS":49152}}' '{"_env":{"CBM_B200_BAND_COLS":24576}}' '{"_env":{"CBM_B200_BAND_COLS":98304}}' > gpurun_out/r18_cfg2_band.jsonl 2> gpurun_out/r18_cfg2_band.err
REPS=20 timeout 600 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_FIXED_TILES":1,"CBM_B200_BAND_COLS":0}}' '{"_env":{"CBM_B200_DENSE_FIXED_TILES":0}}' > gpurun_out/r18_cfg3_tiles.jsonl 2> gpurun_out/r18_cfg3_tiles.err
unset CBM_B200_BAND_COLS
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum -k regex:cbm_kernel -s 1 -c 1 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r18_ncu_cfg4_band.txt 2>&1
timeout 60 ./tools/umma_probe_bf16 > gpurun_out/r18_umma_bf16.txt 2>&1; echo "probe rc=$?" >> gpurun_out/r18_umma_bf16.txt
