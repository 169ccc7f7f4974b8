timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_v6.log 2>&1; echo rc=$? >> gpurun_out/pytest_v6.log
timeout 300 python bench.py --steps 2 --warmup 1 --frames 64 --iters 20 --distinct 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_v6.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1g.csv $CMD > gpurun_out/launch_run7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vn_tile64 -s 2 -c 1 -o gpurun_out/prof_vn_r1g $CMD > gpurun_out/prof_vn7.log 2>&1
