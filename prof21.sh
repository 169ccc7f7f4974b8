timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v14.log 2>&1; echo rc=$? >> gpurun_out/pytest_v14.log
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups 1 >> gpurun_out/bench_v14.log 2>&1; done
timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups 1 --rule lut >> gpurun_out/bench_v14.log 2>&1
