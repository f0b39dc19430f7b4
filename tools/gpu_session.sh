cd $GRAFT_REPO_ROOT
timeout 300 python tools/device_step_profile.py > gpurun_out/r27_devstep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r27_launches.csv python tools/device_step_profile.py > gpurun_out/r27_ncu.log 2>&1
