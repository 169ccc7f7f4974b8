set -x
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv $CMD > gpurun_out/launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cn_update -s 2 -c 2 -o gpurun_out/prof_cn_r1a $CMD > gpurun_out/prof_cn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vn_update -s 1 -c 1 -o gpurun_out/prof_vn_r1a $CMD > gpurun_out/prof_vn.log 2>&1
ls -la gpurun_out
