cd $GRAFT_REPO_ROOT
NOCHECK=1 REPS=3 CBM_B200_DENSE_TRACE=gpurun_out/r13_trace.txt timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' > gpurun_out/r13_cfg3.jsonl 2> gpurun_out/r13_cfg3.err
NOCHECK=1 REPS=3 CBM_B200_DENSE_TRACE=gpurun_out/r13_trace7.txt CBM_B200_DENSE_DBG=15 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' > gpurun_out/r13_cfg3_7.jsonl 2> gpurun_out/r13_cfg3_7.err
