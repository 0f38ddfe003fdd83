cd $GRAFT_REPO_ROOT
NOCHECK=1 REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":1}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":2}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":4}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":3}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":6}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":5}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":7}}' > gpurun_out/r6_cfg3_dbg.jsonl 2> gpurun_out/r6_cfg3_dbg.err
REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":0}}' > gpurun_out/r6_cfg3.jsonl 2> gpurun_out/r6_cfg3.err
timeout 600 python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_kernel" -s 1 -c 1 -o gpurun_out/r6_cfg3_dense python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r6_ncu.log 2>&1
