#!/bin/bash
set -x
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/fer_sweep.py --family r0.1de --snrs 0.155,0.158,0.161,0.163,0.165,0.17 --frames 1024 --out $O/c5_r01de.jsonl > $O/c5.log 2>&1
timeout 600 python bench.py --family r0.1de --no-cpu-baseline > $O/bench_r01de_exact.json 2> $O/bench_r01de_exact.err
timeout 600 python bench.py --family r0.1de --msg-bits 16 --no-cpu-baseline > $O/bench_r01de_exact_m16.json 2> $O/bench_r01de_m16.err
