# Round checks with the current defaults: smoke, pytest -m gpu, both bench arms, ncu launch list + full capture.
cd $GRAFT_REPO_ROOT
bash tools/run_round.sh
