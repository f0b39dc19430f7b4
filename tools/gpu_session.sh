set -x
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/r21_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r21_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r21_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r21_bench.json 2> gpurun_out/r21_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r21_ref.json 2> gpurun_out/r21_ref.err
