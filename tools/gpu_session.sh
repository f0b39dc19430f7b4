cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_bench.py -q -p no:cacheprovider -x > gpurun_out/r37_bench_test.log 2>&1; echo "rc=$?" >> gpurun_out/r37_bench_test.log
