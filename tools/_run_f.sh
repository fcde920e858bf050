cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02c_gputest.txt
python bench.py > gpurun_out/r02c_bench_C2.json 2> gpurun_out/r02c_bench_C2.err
python bench.py --config C4 --no-cpu > gpurun_out/r02c_bench_C4.json 2> gpurun_out/r02c_bench_C4.err
python bench.py --config C1 > gpurun_out/r02c_bench_C1.json 2> gpurun_out/r02c_bench_C1.err
