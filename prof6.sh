timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v5.log 2>&1; echo rc=$? >> gpurun_out/pytest_v5.log
timeout 300 python bench.py --steps 2 --warmup 1 --frames 64 --iters 20 --distinct 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_v5.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 1 --frames 64 --iters 20 --distinct 8 --no-e2e --no-cpu-baseline --rule lut > gpurun_out/bench_v5_lut.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cn_tile -s 3 -c 1 -o gpurun_out/prof_cn_r1e $CMD > gpurun_out/prof_cn5.log 2>&1
