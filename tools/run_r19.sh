# Secondary bench lines on the other small configs (C1, C3) with the current defaults.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?" >> gpurun_out/bench_c1.err
timeout 600 python bench.py --config 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?" >> gpurun_out/bench_c3.err
