set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu2.log
timeout 600 python bench.py --steps 3 --warmup 2 --frames 128 --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv $CMD > gpurun_out/launch_run2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cn_tile -s 3 -c 3 -o gpurun_out/prof_cn_r1b $CMD > gpurun_out/prof_cn2.log 2>&1
