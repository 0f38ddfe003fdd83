cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CBM_B200_DENSE_TRACE=gpurun_out/r30_trace_full.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 '{}' > /dev/null 2> gpurun_out/r30_trace.err
CBM_B200_DENSE_TRACE=gpurun_out/r30_trace_skel.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":15}}' > /dev/null 2>> gpurun_out/r30_trace.err
python tools/trace_dense.py gpurun_out/r30_trace_full.txt > gpurun_out/r30_trace_full_summary.txt 2>&1
python tools/trace_dense.py gpurun_out/r30_trace_skel.txt > gpurun_out/r30_trace_skel_summary.txt 2>&1
