cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --legs main,bf16 > gpurun_out/r53_bench.log 2> gpurun_out/r53_bench.err; echo "rc=$?" >> gpurun_out/r53_bench.err
timeout 900 python -m pytest tests/test_gpu_bench.py -q -p no:cacheprovider > gpurun_out/r53_bt.log 2>&1; echo "rc=$?" >> gpurun_out/r53_bt.log
