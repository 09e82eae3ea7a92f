# GPU setup components + 16-bit column index check (one gpurun session).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_setup.py tests/test_cli.py -q -m gpu > gpurun_out/pytest_setup.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_setup.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "variants or spmv or vcycle or pcg_c1" > gpurun_out/pytest_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
timeout 1200 python tools/tune_kernels.py --sets i16= i32=idx16:0 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
timeout 1500 python tools/setup_timing.py --configs 2,3 --out gpurun_out/setup_timing.json > gpurun_out/setup_timing.log 2>&1
echo "timing rc=$?" >> gpurun_out/setup_timing.log
