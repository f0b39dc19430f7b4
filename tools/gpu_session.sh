cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_device_schedule.py tests/test_gpu_graphs.py -q -p no:cacheprovider > gpurun_out/r55_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r55_devsched.log
for i in 1 2; do timeout 300 python tools/device_step_profile.py >> gpurun_out/r55_devstep.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r55_launches_dev.csv python tools/device_step_profile.py > gpurun_out/r55_ncu_dev.log 2>&1
