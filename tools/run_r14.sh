# Long-row split for CSR operands + collapsed dense coarse tail: parity tests, then a tune sweep on C2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "csr_long or csr_kernel_variants or dense_coarse" > gpurun_out/pytest_r14.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r14.log
timeout 1500 python tools/tune_kernels.py --sets base= long2=csr_long:2 long4=csr_long:4 long8=csr_long:8 long2pt2=csr_long:2,csr_per_thread:2 td1500=tail_dense:1500 td7000=tail_dense:7000 td1500l4=tail_dense:1500,csr_long:4 > gpurun_out/tune_r14.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r14.log
timeout 600 python tools/tune_kernels.py --config 1 --sets base= td1500=tail_dense:1500 td6000=tail_dense:6000 long4=csr_long:4 --out gpurun_out/tune_c1.json > gpurun_out/tune_r14_c1.log 2>&1
echo "tune c1 rc=$?" >> gpurun_out/tune_r14_c1.log
