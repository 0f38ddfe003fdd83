cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in libcbm_b200.so libcbm_b200_altA.so libcbm_b200_altB.so libcbm_b200_altC.so libcbm_b200.so; do
  echo "== $lib" >> gpurun_out/r27_cfg3_dense_roles.jsonl
  CBM_B200_LIB=$lib REPS=20 timeout 600 python tools/time_workload.py cfg3 '{}' '{"_env":{"CBM_B200_DENSE_DBG":15}}' >> gpurun_out/r27_cfg3_dense_roles.jsonl 2>> gpurun_out/r27_cfg3_dense_roles.err
done
