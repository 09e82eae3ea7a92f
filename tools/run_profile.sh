#!/bin/bash
# ncu evidence for EVERY launch of one PCG iteration (GPU box, one GPU):
#   tools/run_profile.sh <config> <tag> [profile_iter options...]
# 1. plain run (must exit 0 without ncu) -> the op table (one line per launch, in order)
# 2. launch list: gpu__time_duration.sum of every launch of the profiled iteration
# 3. --set full capture of the same launches (all ops, not a subset), exported as a raw CSV
#    next to the .ncu-rep (the rep itself is kept only when it fits gpurun_out's budget)
# tools/ncu_summary.py turns the CSVs into profiles/ncu_<tag>_*.csv here.
CFG=${1:-2}; TAG=${2:-r02}; shift 2
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
O=gpurun_out/prof_${TAG}
python tools/profile_iter.py --config $CFG "$@" > ${O}_plain.log 2>&1 || { echo "plain run failed"; tail -5 ${O}_plain.log; exit 1; }
NOPS=$(grep -cE " L[0-9]+ +[0-9.]+ us" ${O}_plain.log)
echo "ops per iteration: $NOPS"
# profile_iter runs the body twice between cuProfilerStart/Stop: skip the warm pass
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    -s $NOPS -c $NOPS --log-file ${O}_launches.csv python tools/profile_iter.py --config $CFG "$@" > ${O}_ncu_list.log 2>&1
echo "list rc=$?"
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -s $NOPS -c $NOPS -f -o ${O}_full python tools/profile_iter.py --config $CFG "$@" > ${O}_ncu_full.log 2>&1
echo "full rc=$?"
ncu -i ${O}_full.ncu-rep --page raw --csv > ${O}_full_raw.csv 2> /dev/null
ls -la ${O}_full.ncu-rep
# keep the report only if small enough to travel back with everything else
SZ=$(stat -c %s ${O}_full.ncu-rep 2>/dev/null || echo 0)
if [ "$SZ" -gt 30000000 ]; then rm -f ${O}_full.ncu-rep; echo "rep dropped ($SZ bytes); raw CSV kept"; fi
