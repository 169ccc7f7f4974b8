timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v9.log 2>&1; echo rc=$? >> gpurun_out/pytest_v9.log
timeout 600 python bench.py > gpurun_out/bench_v9.log 2>&1
timeout 600 python bench.py --frames 512 --groups 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_v9_512.log 2>&1
