cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py tests/test_gpu_parity.py -q -m gpu -k "matrix_market or variants" > gpurun_out/pytest_fix.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_fix.log
timeout 1500 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
timeout 1200 python tools/tune_kernels.py --sets i32a=idx16:0 i16a= i32b=idx16:0 i16b= > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
