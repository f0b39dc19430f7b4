cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/r32_bench.log 2> gpurun_out/r32_bench.err; echo "rc=$?" >> gpurun_out/r32_bench.err
timeout 600 python -m pytest tests/test_gpu_device_schedule.py -q -p no:cacheprovider > gpurun_out/r32_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r32_devsched.log
timeout 3000 python tools/kernel_mutation.py run > gpurun_out/r32_mutation.log 2>&1; echo "rc=$?" >> gpurun_out/r32_mutation.log
timeout 600 python tools/diag_rw43.py > gpurun_out/r32_rw43.log 2>&1; echo "rc=$?" >> gpurun_out/r32_rw43.log
