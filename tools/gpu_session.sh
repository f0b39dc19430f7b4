cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 600 python bench.py --legs main > gpurun_out/r42_bench$i.log 2> gpurun_out/r42_bench$i.err; done
