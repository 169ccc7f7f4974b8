#!/bin/bash
# GPU call: validation of the pruned round-2 code: full suite, smoke, bench lines, production-graph DRAM traffic, sanitizers
set -x
O=gpurun_out/r2r; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --msg-bits 16 --no-cpu-baseline > $O/bench_m16.json 2> $O/bench_m16.err
timeout 900 python bench.py --rule lut --msg-bits 16 --no-cpu-baseline > $O/bench_lut_m16.json 2> $O/bench_lut_m16.err
timeout 900 python bench.py --no-et --no-cpu-baseline > $O/bench_noet.json 2> $O/bench_noet.err
timeout 900 ncu --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/graph_traffic.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 20 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9 --num-cuda-barriers 4096"
for t in memcheck racecheck synccheck; do
  METLDPC_GRAPH=0 timeout 900 $SAN --tool $t python tools/sanitize_c1.py > $O/sanitize_${t}_graph0.log 2>&1; echo "rc=$?" >> $O/sanitize_${t}_graph0.log
done
