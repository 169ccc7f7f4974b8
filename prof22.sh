CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 6 --distinct 8 --no-e2e --no-cpu-baseline --groups 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cn_tile -s 3 -c 1 -o gpurun_out/prof_r1m $CMD > gpurun_out/prof_r1m.log 2>&1
