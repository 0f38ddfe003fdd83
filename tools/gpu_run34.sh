cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for dbg in 0 64 128 192 4 12 132 140 141; do
  rm -f /tmp/tr.txt
  CBM_B200_DENSE_TRACE=/tmp/tr.txt NOCHECK=1 REPS=1 timeout 600 python tools/time_workload.py cfg3 "{\"_env\":{\"CBM_B200_DENSE_DBG\":$dbg}}" > /dev/null 2>> gpurun_out/r34.err
  echo "== DBG=$dbg" >> gpurun_out/r34_mma_issue.txt
  python tools/trace_dense.py /tmp/tr.txt 2>&1 | head -4 >> gpurun_out/r34_mma_issue.txt
done
