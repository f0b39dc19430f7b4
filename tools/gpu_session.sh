set -x
cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_rw43.py > gpurun_out/r11_rw43.log 2>&1
timeout 900 python bench.py > gpurun_out/r11_bench.json 2> gpurun_out/r11_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r11_launches.csv python bench.py --steps 5 --warmup 3 --legs main,probe,bf16,p2p > gpurun_out/r11_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grass_stream_kernel -s 3 -c 1 -o gpurun_out/r11_k2 python bench.py --steps 3 --warmup 3 --legs main > gpurun_out/r11_ncu_k2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grass_stream_kernel -s 2 -c 1 -o gpurun_out/r11_k1bf16 python tools/k1_bf16_probe.py > gpurun_out/r11_ncu_k1.log 2>&1
