cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs 2>&1 | tail -15 > gpurun_out/r02d_gputest.txt
python bench.py > gpurun_out/r02d_bench_C2.json 2> gpurun_out/r02d_bench_C2.err
python bench.py --config C4 --no-cpu > gpurun_out/r02d_bench_C4.json 2> gpurun_out/r02d_bench_C4.err
python bench.py --impl reference > gpurun_out/r02d_ref_C2.json 2> gpurun_out/r02d_ref_C2.err
nproc > gpurun_out/r02d_nproc.txt; lscpu | head -20 >> gpurun_out/r02d_nproc.txt
