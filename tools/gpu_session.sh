cd $GRAFT_REPO_ROOT
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none --import-source on -k regex:grass_finalize -s 5 -c 1 -o gpurun_out/r45_k3 python tools/device_step_profile.py > gpurun_out/r45_ncu_k3.log 2>&1
timeout 900 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none --import-source on -k regex:grass_commit -c 1 -o gpurun_out/r45_cm python tools/device_step_profile.py > gpurun_out/r45_ncu_cm.log 2>&1
