cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 600 > gpurun_out/r51_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r51_gpu_tests.log
for i in 1 2; do timeout 300 python tools/device_step_profile.py >> gpurun_out/r51_devstep.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r51_launches_dev.csv python tools/device_step_profile.py > gpurun_out/r51_ncu_dev.log 2>&1
timeout 600 python bench.py --legs main,probe > gpurun_out/r51_bench.log 2> gpurun_out/r51_bench.err
