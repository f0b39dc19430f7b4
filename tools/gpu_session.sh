cd $GRAFT_REPO_ROOT
timeout 3000 python tools/kernel_mutation.py run > gpurun_out/r60_mutation.log 2>&1; echo "rc=$?" >> gpurun_out/r60_mutation.log
