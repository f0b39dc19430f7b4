set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 500 python tools/dbg_nccl_a2a.py > gpurun_out/r3_nccl.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest.log
GRASS_RECORD_DIR=gpurun_out timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "zero_theta_update" -p no:cacheprovider > gpurun_out/r3_r21.log 2>&1
timeout 1200 python tools/variants.py run > gpurun_out/r3_variants.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grass_stream_kernel -s 2 -c 1 -o gpurun_out/r3_k1bf16 python tools/k1_bf16_probe.py > gpurun_out/r3_ncu.log 2>&1
