cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=12 timeout 2400 python tools/time_workload.py cfg4_b256 '{}' '{"split_threshold":128,"chunk":32}' '{"split_threshold":128,"chunk":64}' '{"split_threshold":256,"chunk":128}' '{"split_threshold":512,"chunk":64}' '{"split_threshold":512,"chunk":128}' '{"split_threshold":1024,"chunk":128}' '{"split_threshold":1024,"chunk":256}' '{}' > gpurun_out/r46_cfg4_split.jsonl 2> gpurun_out/r46_cfg4_split.err
