set -x
cd $GRAFT_REPO_ROOT
timeout 2400 python tools/kernel_mutation.py run > gpurun_out/r16_mutation.log 2>&1
timeout 900 python bench.py --model llama3-8b --gamma 4 --legs main,probe,bf16,offload --steps 20 > gpurun_out/r16_bench_8b.json 2> gpurun_out/r16_bench_8b.err
timeout 1500 python tools/bench_13b_offload.py > gpurun_out/r16_13b.json 2> gpurun_out/r16_13b.err
