cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > gpurun_out/r3_dense_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r3_dense_tests.log
REPS=10 timeout 900 python tools/time_workload.py cfg3 '{"dense":0}' '{"dense":1}' '{"dense":1,"dense_min":2}' '{"dense":1,"dense_min":6}' > gpurun_out/r3_cfg3.jsonl 2> gpurun_out/r3_cfg3.err
REPS=10 timeout 900 python tools/time_workload.py cfg2 '{"dense":0}' '{"dense":1}' '{"dense":1,"dense_min":2}' > gpurun_out/r3_cfg2.jsonl 2> gpurun_out/r3_cfg2.err
REPS=10 timeout 900 python tools/time_workload.py cfg0 '{"dense":0}' '{"dense":1}' > gpurun_out/r3_cfg0.jsonl 2> gpurun_out/r3_cfg0.err
REPS=10 timeout 900 python tools/time_workload.py cfg1 '{"dense":0}' '{"dense":1}' > gpurun_out/r3_cfg1.jsonl 2> gpurun_out/r3_cfg1.err
