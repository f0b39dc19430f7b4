cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grass_stream_kernel -s 3 -c 1 -o gpurun_out/r36_k2dev python tools/device_step_profile.py > gpurun_out/r36_ncu_k2.log 2>&1; echo "rc=$?" >> gpurun_out/r36_ncu_k2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grass_commit_sample -s 3 -c 1 -o gpurun_out/r36_commit python tools/device_step_profile.py > gpurun_out/r36_ncu_commit.log 2>&1; echo "rc=$?" >> gpurun_out/r36_ncu_commit.log
