cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/r5_dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r5_dense_tests.log
REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":1}' > gpurun_out/r5_cfg3.jsonl 2> gpurun_out/r5_cfg3.err
timeout 600 python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_cfg3_launches.csv python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r5_ncu_list.log 2>&1
REPS=10 timeout 900 python tools/time_workload.py cfg2 '{"dense":0}' '{"dense":1}' '{"dense":1,"dense_min":2}' > gpurun_out/r5_cfg2.jsonl 2> gpurun_out/r5_cfg2.err
REPS=5 timeout 1200 python tools/time_workload.py cfg4_b256 '{"dense":0}' '{"dense":1}' '{"dense":1,"dense_min":2}' > gpurun_out/r5_cfg4.jsonl 2> gpurun_out/r5_cfg4.err
