#!/bin/bash
# GPU call: C5 sweep of the density-evolution stand-in r0.1de, bench at the headline config, synccheck
set -x
O=gpurun_out/r2e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/fer_sweep.py --family r0.1de --snrs 0.15,0.155,0.158,0.161,0.165,0.17,0.18 --frames 1024 --out $O/c5_r01de.jsonl > $O/c5.log 2>&1
timeout 600 python bench.py --family r0.1de > $O/bench_r01de_exact.json 2> $O/bench_r01de_exact.err
timeout 600 python bench.py --family r0.1de --msg-bits 16 --no-cpu-baseline > $O/bench_r01de_exact_m16.json 2> $O/bench_r01de_m16.err
timeout 600 python bench.py --family r0.1de --no-refill --no-cpu-baseline --no-e2e > $O/bench_r01de_group.json 2> $O/bench_r01de_group.err
METLDPC_GRAPH=0 timeout 900 compute-sanitizer --print-limit 20 --error-exitcode 9 --num-cuda-barriers 4096 --tool synccheck python tools/sanitize_c1.py > $O/sanitize_synccheck_graph0.log 2>&1; echo "rc=$?" >> $O/sanitize_synccheck_graph0.log
