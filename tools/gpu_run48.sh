cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=12 timeout 2400 python tools/time_workload.py cfg4_b256 '{}' '{"split_threshold":2048,"chunk":256}' '{"split_threshold":2048,"chunk":512}' '{"split_threshold":4096,"chunk":256}' '{"split_threshold":1024,"chunk":512}' '{"split_threshold":1024,"chunk":128}' '{}' > gpurun_out/r48_cfg4_split.jsonl 2> gpurun_out/r48_cfg4_split.err
REPS=20 timeout 600 python tools/time_workload.py cfg2 '{}' '{"split_threshold":512,"chunk":128}' '{"split_threshold":1024,"chunk":256}' '{"split_threshold":128,"chunk":32}' '{}' > gpurun_out/r48_cfg2_split.jsonl 2> gpurun_out/r48_cfg2_split.err
