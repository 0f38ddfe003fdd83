cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NOCHECK=1 REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":16}}' '{"_env":{"CBM_B200_DENSE_DBG":32}}' '{"_env":{"CBM_B200_DENSE_DBG":31}}' '{"_env":{"CBM_B200_DENSE_DBG":48}}' > gpurun_out/r28_cfg3_split.jsonl 2> gpurun_out/r28_cfg3_split.err
CBM_B200_DENSE_TRACE=gpurun_out/r28_dense_trace.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 '{}' > /dev/null 2> gpurun_out/r28_trace.err
