cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":512}}' '{"_env":{"CBM_B200_DENSE_DBG":32}}' '{"_env":{"CBM_B200_DENSE_DBG":544}}' > gpurun_out/r40_cfg3.jsonl 2> gpurun_out/r40_cfg3.err
