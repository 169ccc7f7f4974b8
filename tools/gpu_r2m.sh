#!/bin/bash
# GPU call: final r0.1de (one core class) + CW 23 ring: full suite, smoke, bench lines, C5 sweeps, ncu of the CN classes
set -x
O=gpurun_out/r2m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --msg-bits 16 --no-cpu-baseline > $O/bench_m16.json 2> $O/bench_m16.err
timeout 900 python bench.py --rule lut --msg-bits 16 --no-cpu-baseline > $O/bench_lut_m16.json 2> $O/bench_lut_m16.err
timeout 900 python bench.py --no-et --no-cpu-baseline > $O/bench_noet.json 2> $O/bench_noet.err
timeout 900 python bench.py --input md --no-cpu-baseline > $O/bench_md.json 2> $O/bench_md.err
timeout 900 python tools/fer_sweep.py --family r0.1de --channel biawgn --snrs 0.15,0.153,0.155,0.158,0.161,0.165,0.17 --frames 2048 --out $O/c5_biawgn.jsonl > $O/c5b.log 2>&1
timeout 900 python tools/fer_sweep.py --family r0.1de --channel md --snrs 0.161,0.165,0.168,0.17,0.175,0.18 --frames 2048 --out $O/c5_md.jsonl > $O/c5m.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring" --launch-skip 3 -c 3 -o $O/ring_default python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu_ring.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_noet.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 20 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
