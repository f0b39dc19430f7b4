cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_device_schedule.py -q -p no:cacheprovider > gpurun_out/r49_devsched.log 2>&1; echo "rc=$?" >> gpurun_out/r49_devsched.log
for v in base k3_nosampler; do
  GRASS_LIB_PATH=build/variants/libgrass_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r49_$v.csv python tools/device_step_profile.py > gpurun_out/r49_$v.log 2>&1
  GRASS_LIB_PATH=build/variants/libgrass_$v.so timeout 300 python tools/device_step_profile.py >> gpurun_out/r49_$v.log 2>&1
done
