cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --model llama3-8b --gamma 4 > gpurun_out/r47_bench_8b.log 2> gpurun_out/r47_bench_8b.err; echo "rc=$?" >> gpurun_out/r47_bench_8b.err
