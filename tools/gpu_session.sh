cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r54_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r54_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/r54_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r54_smoke.log
timeout 600 python bench.py > gpurun_out/r54_bench.log 2> gpurun_out/r54_bench.err; echo "rc=$?" >> gpurun_out/r54_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r54_ref.log 2> gpurun_out/r54_ref.err; echo "rc=$?" >> gpurun_out/r54_ref.err
