# CSR variants (8 loads per round, row-pointer prefetch): bit-identity tests, then a tune sweep on C2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "csr_kernel_variants or rseg" > gpurun_out/pytest_r11.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r11.log
timeout 1500 python tools/tune_kernels.py --sets base= pf=csr_pf:1 u8all=csr_u8:2 u8pf=csr_u8:2,csr_pf:1 u8l=csr_u8:1 pfs256=csr_pf:1,sell_sort:1,sell_sigma:256 > gpurun_out/tune_r11.log 2>&1
echo "tune rc=$?" >> gpurun_out/tune_r11.log
