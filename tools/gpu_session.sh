cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_device_schedule.py -q -p no:cacheprovider > gpurun_out/r39_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r39_devsched.log
timeout 300 python tools/device_step_profile.py > gpurun_out/r39_devstep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r39_launches.csv python tools/device_step_profile.py > gpurun_out/r39_ncu.log 2>&1
