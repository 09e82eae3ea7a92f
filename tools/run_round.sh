#!/bin/bash
# One GPU session in the driver's order (tests, smoke, reference arm, GPU arm) on a
# cold box, then the ncu evidence for every launch of one iteration on C5 and C2.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out
TAG=${TAG:-r02}
STEPS="${1:-tests smoke c5ref c5 prof5 prof2 c2 asm}"
{ nvidia-smi; free -g; nproc; lscpu | grep "Model name"; } > $O/box_d.txt 2>&1
for s in $STEPS; do
  t0=$(date +%s)
  case $s in
    tests) timeout 2400 python -m pytest tests/ -q -m gpu --durations=8 > $O/pytest_gpu_d.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_d.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_d.log 2>&1; echo "smoke rc=$?" >> $O/smoke_d.log ;;
    c5ref) timeout 2400 python bench.py --impl reference > $O/bench_${TAG}_c5_reference.json 2> $O/bench_c5_ref_d.err; echo "rc=$?" >> $O/bench_c5_ref_d.err ;;
    c5) timeout 2400 python bench.py > $O/bench_${TAG}_c5.json 2> $O/bench_c5_d.err; echo "rc=$?" >> $O/bench_c5_d.err ;;
    c2) timeout 900 python bench.py --config 2 > $O/bench_${TAG}_c2.json 2> $O/bench_c2_d.err; echo "rc=$?" >> $O/bench_c2_d.err
        timeout 900 python bench.py --config 2 --impl reference > $O/bench_${TAG}_c2_reference.json 2>> $O/bench_c2_d.err ;;
    prof5) timeout 2400 bash tools/run_profile.sh 5 ${TAG}_c5 > $O/prof5_d.log 2>&1 ;;
    prof2) timeout 1500 bash tools/run_profile.sh 2 ${TAG}_c2 > $O/prof2_d.log 2>&1 ;;
    asm) timeout 900 python tools/time_assembly.py > $O/assembly_${TAG}.json 2> $O/asm_d.err ;;
  esac
  echo "$s: $(( $(date +%s) - t0 )) s" >> $O/steps_d.txt
done
