cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BENCH_DEV_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config cfg2 --steps 5 --no-cpu-baseline --no-north-star > gpurun_out/r41_share2_cfg2.json 2> gpurun_out/r41_share2.err; echo "share2 rc=$?" >> gpurun_out/r41_share2.err
BENCH_DEV_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --config cfg2 --row-groups 1 --steps 5 --no-cpu-baseline --no-north-star > gpurun_out/r41_share2_cfg2_cols.json 2>> gpurun_out/r41_share2.err; echo "share2 cols rc=$?" >> gpurun_out/r41_share2.err
timeout 900 python bench.py --config cfg2 --steps 10 > gpurun_out/r41_bench_cfg2.json 2> gpurun_out/r41_bench_cfg2.err; echo "cfg2 rc=$?" >> gpurun_out/r41_bench_cfg2.err
