timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v12.log 2>&1; echo rc=$? >> gpurun_out/pytest_v12.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_v12.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 6 --distinct 8 --no-e2e --no-cpu-baseline --groups 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1j.csv $CMD > gpurun_out/launch_run12.log 2>&1
