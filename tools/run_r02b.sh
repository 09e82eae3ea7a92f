#!/bin/bash
# Round-2 GPU session B: tests with the corrected defaults, C5 / C2 option sweeps, C5 oracle fixture.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
STEPS="${1:-tests tune5 golden5 tune2}"
for s in $STEPS; do
  t0=$(date +%s)
  case $s in
    tests) ASPAMG_TEST_C5=0 timeout 1800 python -m pytest tests/ -q -m gpu --durations=12 > $O/pytest_gpu_b.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_b.log ;;
    tune5) timeout 2400 python tools/tune_kernels.py --config 5 --solves 1 --out $O/tune_c5_b.json --sets default= cpt5=csr_per_thread:5 cpt8=csr_per_thread:8 pf2=csr_pf:2 pf2cpt8=csr_pf:2,csr_per_thread:8 fuse_rr=fuse_rr:1 keep96=keep_bytes:100663296 xsellGt=xsell:4 i16g64=idx16_max_group:64 > $O/tune_c5_b.log 2>&1 ;;
    golden5) timeout 2400 python tools/make_full_golden.py --config 5 --out $O/c5_oracle.npz > $O/golden5.log 2>&1 ;;
    tune2) timeout 900 python tools/tune_kernels.py --config 2 --out $O/tune_c2_b.json --sets default= cpt5=csr_per_thread:5 cpt8=csr_per_thread:8 pf2=csr_pf:2 fuse_rr=fuse_rr:1 keep96=keep_bytes:100663296 xsellGt=xsell:4 i16g64=idx16_max_group:64 > $O/tune_c2_b.log 2>&1 ;;
  esac
  echo "$s: $(( $(date +%s) - t0 )) s" >> $O/steps_b.txt
done
