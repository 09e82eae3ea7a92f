cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "not c2_full" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/tune_kernels.py --sets pipe= nopipe=csr_pipe:0 > gpurun_out/tune.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune.log
