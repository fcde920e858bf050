cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/reference_suite.log
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 2>&1 | tail -30 > gpurun_out/r02e_gputest.txt
