#!/bin/bash
# GPU call: full suite + smoke on the round-2 defaults, bench lines, ncu of the headline CN kernel
set -x
O=gpurun_out/r2k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --msg-bits 16 --no-cpu-baseline > $O/bench_m16.json 2> $O/bench_m16.err
timeout 900 python bench.py --rule lut --msg-bits 16 --no-cpu-baseline > $O/bench_lut_m16.json 2> $O/bench_lut_m16.err
timeout 900 python bench.py --input md --no-cpu-baseline > $O/bench_md.json 2> $O/bench_md.err
timeout 900 python bench.py --family r0.1 --input md --no-cpu-baseline --frames 256 > $O/bench_r01_md.json 2> $O/bench_r01_md.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring" --launch-skip 6 -c 3 -o $O/ring_default python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu_ring.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 2000 -c 600 --csv --log-file $O/launches_refill.csv python bench.py --steps 1 --warmup 0 --frames 512 --no-cpu-baseline --no-e2e > /dev/null 2>&1
