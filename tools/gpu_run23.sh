cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=12 timeout 1800 python tools/time_workload.py cfg4_b256 '{"_env":{"CBM_B200_NO_ROW_KEYS":1}}' '{"_env":{"CBM_B200_NO_ROW_KEYS":0}}' '{"_env":{"CBM_B200_BAND_COLS":24576}}' '{"_env":{"CBM_B200_BAND_COLS":32768}}' '{"_env":{"CBM_B200_BAND_COLS":65536}}' > gpurun_out/r23_cfg4_keys.jsonl 2> gpurun_out/r23_cfg4_keys.err
unset CBM_B200_BAND_COLS CBM_B200_NO_ROW_KEYS
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{"_env":{"CBM_B200_NO_ROW_KEYS":1}}' '{"_env":{"CBM_B200_NO_ROW_KEYS":0}}' > gpurun_out/r23_cfg2_keys.jsonl 2> gpurun_out/r23_cfg2_keys.err
unset CBM_B200_NO_ROW_KEYS
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum -k regex:'cbm_kernel|dense_kernel|hub_reduce' -s 5 -c 5 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r23_ncu_cfg4.txt 2>&1
