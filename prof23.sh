timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_full_r1b.log 2>&1; echo rc=$? >> gpurun_out/pytest_full_r1b.log
timeout 600 python bench.py > gpurun_out/bench_full_r1b.log 2>&1
timeout 600 python bench.py --rule lut --no-cpu-baseline > gpurun_out/bench_full_lut_r1b.log 2>&1
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --distinct 8 --no-e2e --no-cpu-baseline --groups 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1n.csv $CMD > gpurun_out/launch_run_r1n.log 2>&1
CMD2="python bench.py --steps 1 --warmup 0 --frames 64 --iters 6 --distinct 8 --no-e2e --no-cpu-baseline --groups 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cn_tile|k_finish" -s 12 -c 4 -o gpurun_out/prof_r1n $CMD2 > gpurun_out/prof_r1n.log 2>&1
