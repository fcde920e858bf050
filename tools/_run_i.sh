cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/reference_suite.log
timeout 2400 python -m pytest tests -m gpu -q -rs -x 2>&1 | tail -40 > gpurun_out/r02f_gputest.txt
