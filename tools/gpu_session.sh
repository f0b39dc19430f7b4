cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/r31_bench.log 2> gpurun_out/r31_bench.err; echo "rc=$?" >> gpurun_out/r31_bench.err
timeout 3000 python tools/kernel_mutation.py run > gpurun_out/r31_mutation.log 2>&1; echo "rc=$?" >> gpurun_out/r31_mutation.log
