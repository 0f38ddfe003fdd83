cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/r44_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r44_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r44_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r44_smoke.log
timeout 1500 python bench.py > gpurun_out/r44_bench.json 2> gpurun_out/r44_bench.err; echo "bench rc=$?" >> gpurun_out/r44_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r44_ref.json 2> gpurun_out/r44_ref.err; echo "ref rc=$?" >> gpurun_out/r44_ref.err
