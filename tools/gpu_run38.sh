cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r38_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r38_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r38_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r38_smoke.log
timeout 1500 python bench.py > gpurun_out/r38_bench.json 2> gpurun_out/r38_bench.err; echo "bench rc=$?" >> gpurun_out/r38_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r38_ref.json 2> gpurun_out/r38_ref.err; echo "ref rc=$?" >> gpurun_out/r38_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r38_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r38_ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r38_ncu_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cbm_kernel" -s 1 -c 1 -o gpurun_out/r38_cfg4_cbm_full python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r38_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dense_kernel" -s 1 -c 1 -o gpurun_out/r38_cfg4_hub_dense_full python tools/ncu_workload.py cfg4_b256 3 > gpurun_out/r38_ncu_full2.log 2>&1
