#!/bin/bash
# Option sweep on the GPU box (one GPU): per option set the graph solve time and the per-op profile.
#   tools/run_sweep.sh <config> <tag> name=k:v,k:v ...      (an empty set, "default=", is the baseline)
# e.g. gpurun -- 'bash tools/run_sweep.sh 5 blk default= blk=csr_blocked:1 na=csr_noalloc:1'
# Results: gpurun_out/tune_c<config>_<tag>.{json,log}; the round-2 sweeps are kept in profiles/tune_r02_*.
CFG=${1:-2}; TAG=${2:-sweep}; shift 2
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SOLVES=3; [ "$CFG" = "5" ] && SOLVES=1
timeout 3000 python tools/tune_kernels.py --config $CFG --solves $SOLVES --out gpurun_out/tune_c${CFG}_${TAG}.json --sets "$@" \
    > gpurun_out/tune_c${CFG}_${TAG}.log 2>&1
echo "rc=$?"; head -20 gpurun_out/tune_c${CFG}_${TAG}.log
