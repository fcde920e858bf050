cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/reference_suite.log
timeout 2400 python -m pytest tests -m gpu -q -rs -W ignore::paper_1401_4068_b200.engine.SlowPathWarning 2>&1 > gpurun_out/r02g_gputest_full.txt
tail -5 gpurun_out/r02g_gputest_full.txt
