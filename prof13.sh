for cfg in "1 1" "2 2" "2 1" "4 4" "4 2" "4 1"; do
set -- $cfg
METLDPC_GRID_SPLIT=$2 timeout 300 python bench.py --steps 3 --warmup 1 --frames 256 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups $1 > gpurun_out/bench_K$1_S$2.log 2>&1
done
