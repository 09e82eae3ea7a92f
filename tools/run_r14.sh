# Long-row split for CSR operands: parity tests, then a tune sweep on C2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "csr_long or csr_kernel_variants" > gpurun_out/pytest_r14.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r14.log
timeout 1500 python tools/tune_kernels.py --sets base= long1=csr_long:1 long2=csr_long:2 long4=csr_long:4 long2pt2=csr_long:2,csr_per_thread:2 long1pt8=csr_long:1,csr_per_thread:8 > gpurun_out/tune_r14.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r14.log
