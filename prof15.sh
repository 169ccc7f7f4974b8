timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v10.log 2>&1; echo rc=$? >> gpurun_out/pytest_v10.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v10.log 2>&1
