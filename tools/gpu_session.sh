cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_device_schedule.py -q -p no:cacheprovider --timeout 300 > gpurun_out/r29_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r29_devsched.log
timeout 300 python tools/device_step_profile.py > gpurun_out/r29_devstep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r29_launches.csv python tools/device_step_profile.py > gpurun_out/r29_ncu.log 2>&1
