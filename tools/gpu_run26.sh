cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_COLD_SEGS":0}}' '{"_env":{"CBM_B200_COLD_SEGS":1}}' > gpurun_out/r26_cfg3_cold_segs.jsonl 2> gpurun_out/r26_cfg3_cold_segs.err
unset CBM_B200_COLD_SEGS
REPS=12 timeout 1500 python tools/time_workload.py cfg4_b256 '{}' '{"max_segments":1}' > gpurun_out/r26_cfg4_segs.jsonl 2> gpurun_out/r26_cfg4_segs.err
CBM_B200_COLD_SEGS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:'cbm_kernel' -s 2 -c 1 python tools/ncu_workload.py cfg3 3 > gpurun_out/r26_ncu_cfg3_cold1.txt 2>&1
