set -x
cd $GRAFT_REPO_ROOT
timeout 600 python tools/e2e_chunk_sweep.py > gpurun_out/r17_e2e_chunks.log 2>&1
timeout 900 python bench.py --legs main,train --steps 10 > gpurun_out/r17_bench_train.json 2> gpurun_out/r17_bench_train.err
