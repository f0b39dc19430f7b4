set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/k1_layout_probe.py > gpurun_out/r10_layout.log 2>&1
timeout 1200 python tools/variants.py run > gpurun_out/r10_variants.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -x > gpurun_out/r10_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r10_pytest.log
