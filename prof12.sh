timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v8.log 2>&1; echo rc=$? >> gpurun_out/pytest_v8.log
for K in 1 2 3; do
timeout 300 python bench.py --steps 3 --warmup 1 --frames 192 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups $K > gpurun_out/bench_K$K.log 2>&1
done
