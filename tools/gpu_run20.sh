cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=12 timeout 1500 python tools/time_workload.py cfg4_b256 \
 '{"_env":{"CBM_B200_HOT_USE":0}}' \
 '{"_env":{"CBM_B200_HOT_USE":1}}' \
 '{"_env":{"CBM_B200_HOT_USE":2}}' \
 '{"_env":{"CBM_B200_HOT_USE":3}}' \
 '{"_env":{"CBM_B200_HOT_USE":3,"CBM_B200_HOT_L1":12}}' \
 '{"_env":{"CBM_B200_HOT_USE":3,"CBM_B200_HOT_L1":48}}' \
 '{"_env":{"CBM_B200_HOT_USE":3,"CBM_B200_HOT_L1":24,"CBM_B200_HOT_L2":65536}}' \
 '{"_env":{"CBM_B200_HOT_USE":3,"CBM_B200_HOT_L1":24,"CBM_B200_HOT_L2":16384}}' \
 '{"_env":{"CBM_B200_HOT_USE":3,"CBM_B200_HOT_L1":24,"CBM_B200_HOT_L2":32768,"CBM_B200_BAND_COLS":24576}}' \
 > gpurun_out/r20_cfg4_hot.jsonl 2> gpurun_out/r20_cfg4_hot.err
unset CBM_B200_HOT_L1 CBM_B200_HOT_L2 CBM_B200_BAND_COLS
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{"_env":{"CBM_B200_HOT_USE":0}}' '{"_env":{"CBM_B200_HOT_USE":1}}' '{"_env":{"CBM_B200_HOT_USE":1,"CBM_B200_HOT_L1":48}}' > gpurun_out/r20_cfg2_hot.jsonl 2> gpurun_out/r20_cfg2_hot.err
unset CBM_B200_HOT_L1
CBM_B200_HOT_USE=3 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct -k regex:cbm_kernel -s 1 -c 1 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r20_ncu_cfg4_hot3.txt 2>&1
