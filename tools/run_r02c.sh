#!/bin/bash
# Round-2 GPU session C: new-kernel tests, thread-group cap + pipelined warp-per-row CSR sweeps, C4 oracle fixture.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
STEPS="${1:-tests tune5 tune2 golden4}"
SETS="default= maxg32=csr_max_group:32 maxg32w4=csr_max_group:32,csrw:4 maxg32w8=csr_max_group:32,csrw:8 maxg16=csr_max_group:16 w4=csrw:4 maxg32w4cpt2=csr_max_group:32,csrw:4,csr_per_thread:2"
for s in $STEPS; do
  t0=$(date +%s)
  case $s in
    tests) timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "csrw or fused or xsell_operands" > $O/pytest_gpu_c.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_c.log ;;
    tune5) timeout 2400 python tools/tune_kernels.py --config 5 --solves 1 --out $O/tune_c5_c.json --sets $SETS > $O/tune_c5_c.log 2>&1 ;;
    tune2) timeout 900 python tools/tune_kernels.py --config 2 --out $O/tune_c2_c.json --sets $SETS > $O/tune_c2_c.log 2>&1 ;;
    golden4) timeout 1800 python tools/make_full_golden.py --config 4 --cached 0 --out $O/c4_oracle.npz > $O/golden4.log 2>&1 ;;
  esac
  echo "$s: $(( $(date +%s) - t0 )) s" >> $O/steps_c.txt
done
