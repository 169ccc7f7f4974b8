./build/red_bench > gpurun_out/red_bench.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v7.log 2>&1; echo rc=$? >> gpurun_out/pytest_v7.log
timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_v7.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --rule lut > gpurun_out/bench_v7_lut.log 2>&1
