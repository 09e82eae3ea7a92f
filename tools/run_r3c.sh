cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_setup.py -q -m gpu -x > gpurun_out/pytest_setup.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_setup.log
timeout 900 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
timeout 1200 python tools/setup_timing.py --configs 5 --scale 2 --out gpurun_out/setup_timing_c5s2.json > gpurun_out/setup_timing_c5s2.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing_c5s2.log
bash tools/run_ncu_g.sh
timeout 1200 python tools/tune_kernels.py --sets base= u84=sell_u:84 u44=sell_u:44 sort=sell_sort:1 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
