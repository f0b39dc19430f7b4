set -x
cd $GRAFT_REPO_ROOT
timeout 3000 python tools/kernel_mutation.py run > gpurun_out/r20_mutation.log 2>&1
