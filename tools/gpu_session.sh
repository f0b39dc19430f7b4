cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_soak.py -q -p no:cacheprovider > gpurun_out/r61_soak.log 2>&1; echo "rc=$?" >> gpurun_out/r61_soak.log
