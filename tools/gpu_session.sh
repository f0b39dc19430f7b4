cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r62_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r62_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/r62_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r62_smoke.log
