cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r24_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r24_pytest.log
timeout 1500 python bench.py > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err; echo "bench rc=$?" >> gpurun_out/r24_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r24_ref.json 2> gpurun_out/r24_ref.err; echo "ref rc=$?" >> gpurun_out/r24_ref.err
REPS=12 timeout 1200 python tools/time_workload.py cfg4_n256 '{"hub":-1}' '{"hub":0}' > gpurun_out/r24_cfg4_n256.jsonl 2> gpurun_out/r24_cfg4_n256.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum -k regex:'cbm_kernel|dense_kernel' -s 4 -c 2 python tools/ncu_workload.py cfg3 3 > gpurun_out/r24_ncu_cfg3.txt 2>&1
timeout 1500 python tools/project_shards.py cfg4_b256 > gpurun_out/r24_project_cfg4_b256_cols.jsonl 2> gpurun_out/r24_project_cols.err
timeout 1800 python tools/project_shards.py cfg4_b256 --2d > gpurun_out/r24_project_cfg4_b256_2d.jsonl 2> gpurun_out/r24_project_2d.err
