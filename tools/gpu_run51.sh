cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in cfg4_n256 cfg4_b128 cfg4_b64 cfg4_n128 cfg4_n64; do
  REPS=12 timeout 900 python tools/time_workload.py $w '{}' >> gpurun_out/r51_cfg4_family.jsonl 2>> gpurun_out/r51_cfg4_family.err
done
