cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/umma_probe_bf16 > gpurun_out/r25_umma_bf16.txt 2>&1; echo "probe rc=$?" >> gpurun_out/r25_umma_bf16.txt
NOCHECK=1 REPS=20 timeout 900 python tools/time_workload.py cfg3 '{"_env":{"CBM_B200_DENSE_DBG":0}}' '{"_env":{"CBM_B200_DENSE_DBG":1}}' '{"_env":{"CBM_B200_DENSE_DBG":2}}' '{"_env":{"CBM_B200_DENSE_DBG":4}}' '{"_env":{"CBM_B200_DENSE_DBG":8}}' '{"_env":{"CBM_B200_DENSE_DBG":3}}' '{"_env":{"CBM_B200_DENSE_DBG":5}}' '{"_env":{"CBM_B200_DENSE_DBG":6}}' '{"_env":{"CBM_B200_DENSE_DBG":7}}' '{"_env":{"CBM_B200_DENSE_DBG":15}}' > gpurun_out/r25_cfg3_dense_dbg.jsonl 2> gpurun_out/r25_cfg3_dense_dbg.err
