cd $GRAFT_REPO_ROOT
timeout 600 python tools/diag_zero_copy.py > gpurun_out/r35_zc.log 2>&1; echo "rc=$?" >> gpurun_out/r35_zc.log
