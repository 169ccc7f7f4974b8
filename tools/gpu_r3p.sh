#!/bin/bash
# GPU call: validation of the final code: headline bench line, variants, ncu launch list + CN capture, graph traffic, sanitizers
set -x
O=gpurun_out/r3p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --msg-bits 16 --no-cpu-baseline > $O/bench_m16.json 2> $O/bench_m16.err
timeout 900 python bench.py --rule lut --no-cpu-baseline > $O/bench_lut.json 2> $O/bench_lut.err
timeout 900 python bench.py --no-et --no-cpu-baseline > $O/bench_noet.json 2> $O/bench_noet.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_noet.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 20 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring" --launch-skip 3 -c 3 -o $O/ring_default python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu_ring.log 2>&1
timeout 900 ncu --graph-profiling graph --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/graph_traffic.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 20 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9 --num-cuda-barriers 4096"
timeout 1200 $SAN --tool memcheck python tools/sanitize_c1.py > $O/sanitize_memcheck_graph.log 2>&1; echo "rc=$?" >> $O/sanitize_memcheck_graph.log
for t in memcheck racecheck synccheck; do
  METLDPC_GRAPH=0 timeout 900 $SAN --tool $t python tools/sanitize_c1.py > $O/sanitize_${t}_graph0.log 2>&1; echo "rc=$?" >> $O/sanitize_${t}_graph0.log
done
