cd $GRAFT_REPO_ROOT
GRASS_FUZZ=8 timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_p2p.py tests/test_gpu_soak.py -q -p no:cacheprovider --timeout 900 -k "fuzz or soak" > gpurun_out/r24_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/r24_fuzz.log
