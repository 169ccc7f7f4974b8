export METLDPC_LIB=$PWD/build/variants/cur.so
CMD="python bench.py --steps 1 --warmup 0 --frames 64 --iters 4 --distinct 8 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cn_tile -s 3 -c 1 -o gpurun_out/prof_cn_r1c $CMD > gpurun_out/prof_cn3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vn_update -s 2 -c 1 -o gpurun_out/prof_vn_r1c $CMD > gpurun_out/prof_vn3.log 2>&1
