CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1f.csv $CMD > gpurun_out/launch_run6.log 2>&1
