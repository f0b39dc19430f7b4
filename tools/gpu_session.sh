set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_race.py -q -p no:cacheprovider --timeout 300 > gpurun_out/r19_race.log 2>&1; echo "rc=$?" >> gpurun_out/r19_race.log
timeout 1200 python tools/kernel_mutation.py run 17 18 19 > gpurun_out/r19_mut.log 2>&1
