cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/profile_batch_search.py 1024 7 10000 te > gpurun_out/r02i_prof_bs.txt 2>&1
nproc >> gpurun_out/r02i_prof_bs.txt
