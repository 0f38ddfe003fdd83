cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/r17_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r17_pytest.log
timeout 1200 python bench.py > gpurun_out/r17_bench.json 2> gpurun_out/r17_bench.err; echo "bench rc=$?" >> gpurun_out/r17_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r17_ref.json 2> gpurun_out/r17_ref.err; echo "ref rc=$?" >> gpurun_out/r17_ref.err
BENCH_DEV_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config cfg2 --steps 5 --no-cpu-baseline --no-north-star > gpurun_out/r17_share2.json 2> gpurun_out/r17_share2.err; echo "share2 rc=$?" >> gpurun_out/r17_share2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r17_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r17_ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r17_ncu_bench.log
