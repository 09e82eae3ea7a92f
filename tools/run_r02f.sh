#!/bin/bash
# Round-2 GPU session F: k_csrw variants — contiguous row block per CTA, L1-bypassing matrix loads.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
t0=$(date +%s)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "csrw" > $O/pytest_gpu_f.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_f.log
echo "tests: $(( $(date +%s) - t0 )) s" >> $O/steps_f.txt
SETS="default= blk=csr_blocked:1 na=csr_noalloc:1 blkna=csr_blocked:1,csr_noalloc:1 blknaw8=csr_blocked:1,csr_noalloc:1,csrw:8"
t0=$(date +%s)
timeout 2400 python tools/tune_kernels.py --config 5 --solves 1 --out $O/tune_c5_f.json --sets $SETS > $O/tune_c5_f.log 2>&1
echo "tune5: $(( $(date +%s) - t0 )) s" >> $O/steps_f.txt
t0=$(date +%s)
timeout 900 python tools/tune_kernels.py --config 2 --out $O/tune_c2_f.json --sets $SETS > $O/tune_c2_f.log 2>&1
echo "tune2: $(( $(date +%s) - t0 )) s" >> $O/steps_f.txt
