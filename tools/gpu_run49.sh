cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r49_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r49_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r49_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r49_smoke.log
timeout 1500 python bench.py > gpurun_out/r49_bench.json 2> gpurun_out/r49_bench.err; echo "bench rc=$?" >> gpurun_out/r49_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r49_ref.json 2> gpurun_out/r49_ref.err; echo "ref rc=$?" >> gpurun_out/r49_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r49_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r49_ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r49_ncu_bench.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum -k regex:'cbm_kernel|dense_kernel|hub_reduce' -s 4 -c 4 python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r49_ncu_cfg4.txt 2>&1
