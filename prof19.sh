timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v13.log 2>&1; echo rc=$? >> gpurun_out/pytest_v13.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v13.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --rule lut > gpurun_out/bench_v13_lut.log 2>&1
