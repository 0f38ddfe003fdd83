cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/probe_e2e_sweep.py cfg4_b256 default 1 2 4 8 128/128 64/64/64/64 32/64/64/64/32 32/96/96/32 64/128/64 16/48/64/64/48/16 > gpurun_out/r31_e2e_sweep.txt 2> gpurun_out/r31_e2e_sweep.err
