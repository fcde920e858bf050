cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/reference_suite.log
timeout 2400 python -m pytest tests -m gpu -q -rs -W ignore::paper_1401_4068_b200.engine.SlowPathWarning 2>&1 > gpurun_out/r02h_gputest_full.txt
tail -3 gpurun_out/r02h_gputest_full.txt
python tools/time_radius.py 16 > gpurun_out/r02h_radius.json 2>&1
python bench.py --config C3 --shape 1024,7,10000,te --no-cpu > gpurun_out/r02h_c3_small.json 2> gpurun_out/r02h_c3_small.err
