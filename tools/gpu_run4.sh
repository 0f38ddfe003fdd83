cd $GRAFT_REPO_ROOT
timeout 600 python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_cfg3_launches.csv python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r4_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dense_kernel|cbm_kernel" -s 2 -c 2 -o gpurun_out/r4_cfg3_dense python tools/ncu_workload.py cfg3 3 dense=1 > gpurun_out/r4_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r4_ncu.log
REPS=5 timeout 1200 python tools/time_workload.py cfg4_b256 '{}' '{"_slab":16}' '{"_slab":32}' '{"_slab":64}' '{"_slab":128}' > gpurun_out/r4_cfg4_slabs.jsonl 2> gpurun_out/r4_cfg4_slabs.err
