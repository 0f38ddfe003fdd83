cd $GRAFT_REPO_ROOT
NOCHECK=1 REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":8}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":15}}' '{"dense":1,"_env":{"CBM_B200_DENSE_DBG":0}}' > gpurun_out/r12_cfg3.jsonl 2> gpurun_out/r12_cfg3.err
