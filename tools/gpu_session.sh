cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/r34_bench.log 2> gpurun_out/r34_bench.err; echo "rc=$?" >> gpurun_out/r34_bench.err
