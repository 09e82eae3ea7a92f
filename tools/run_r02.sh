#!/bin/bash
# Round-2 GPU session: tests, C2 quick bench + format sweep, C5 bench (both arms), ncu profiles.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
{ nvidia-smi; free -g; df -h . /tmp; nproc; } > $O/box.txt 2>&1
STEPS="${1:-tests c2 c5ref c5 prof2 prof5}"
for s in $STEPS; do
  t0=$(date +%s)
  case $s in
    tests) ASPAMG_TEST_C5=0 timeout 1500 python -m pytest tests/ -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log ;;
    c2) timeout 600 python bench.py --config 2 --steps 3 --no-cpu > $O/bench_c2.json 2> $O/bench_c2.err; echo "rc=$?" >> $O/bench_c2.err
        timeout 900 python tools/tune_kernels.py --config 2 --sets default= xsell0=xsell:0 --out $O/tune_c2_xsell.json > $O/tune_c2_xsell.log 2>&1 ;;
    c5ref) timeout 2400 python bench.py --impl reference > $O/bench_c5_ref.json 2> $O/bench_c5_ref.err; echo "rc=$?" >> $O/bench_c5_ref.err; ls -la .cache >> $O/box.txt ;;
    c5) timeout 2400 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err ;;
    prof2) timeout 1500 bash tools/run_profile.sh 2 r02_c2 > $O/prof2.log 2>&1 ;;
    prof5) timeout 2400 bash tools/run_profile.sh 5 r02_c5 > $O/prof5.log 2>&1 ;;
  esac
  echo "$s: $(( $(date +%s) - t0 )) s" >> $O/steps.txt
done
