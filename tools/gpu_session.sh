cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r56_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r56_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/r56_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r56_smoke.log
timeout 600 python bench.py > gpurun_out/r56_bench.log 2> gpurun_out/r56_bench.err; echo "rc=$?" >> gpurun_out/r56_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r56_ref.log 2> gpurun_out/r56_ref.err; echo "rc=$?" >> gpurun_out/r56_ref.err
timeout 3000 python tools/kernel_mutation.py run > gpurun_out/r56_mutation.log 2>&1; echo "rc=$?" >> gpurun_out/r56_mutation.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r56_launches_dev.csv python tools/device_step_profile.py > gpurun_out/r56_ncu_dev.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r56_launches.csv python bench.py --steps 2 --warmup 3 --legs main > gpurun_out/r56_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grass_stream_kernel -s 3 -c 1 -o gpurun_out/r56_k2dev python tools/device_step_profile.py > gpurun_out/r56_ncu_k2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grass_finalize -s 3 -c 1 -o gpurun_out/r56_k3 python tools/device_step_profile.py > gpurun_out/r56_ncu_k3.log 2>&1
for i in 1 2; do timeout 300 python tools/device_step_profile.py >> gpurun_out/r56_devstep.log 2>&1; done
