cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_device_schedule.py -q -p no:cacheprovider > gpurun_out/r57_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r57_devsched.log
