cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/tune_kernels.py --sets base= pt2=csr_per_thread:2 pt8=csr_per_thread:8 sort256=sell_sort:1,sell_sigma:256 sort64=sell_sort:1,sell_sigma:64 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
timeout 900 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
