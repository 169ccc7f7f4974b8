#!/bin/bash
# GPU call: headline config (r0.1de, BIAWGN input), new parity tests, bench lines, sweeps, CW A/B
set -x
O=gpurun_out/r2i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_paths.py -x -q -k "r01de or headline" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 600 python bench.py --msg-bits 16 --no-cpu-baseline > $O/bench_default_m16.json 2> $O/bench_default_m16.err
timeout 600 python bench.py --no-et --no-cpu-baseline > $O/bench_default_noet.json 2> $O/bench_default_noet.err
timeout 600 python bench.py --input md --no-cpu-baseline > $O/bench_md.json 2> $O/bench_md.err
timeout 600 python bench.py --family r0.1 --input md --no-cpu-baseline --no-e2e > $O/bench_r01_md.json 2> $O/bench_r01_md.err
timeout 900 python tools/fer_sweep.py --family r0.1de --channel biawgn --snrs 0.15,0.153,0.155,0.158,0.161,0.165,0.17 --frames 1024 --out $O/c5_r01de_biawgn.jsonl > $O/c5b.log 2>&1
timeout 900 python tools/fer_sweep.py --family r0.1de --channel md --snrs 0.161,0.165,0.168,0.17,0.175,0.18 --frames 1024 --out $O/c5_r01de_md.jsonl > $O/c5m.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-et --msg-bits 16"
for rep in 1 2; do
  timeout 300 $B > $O/ab_cw31_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$PWD/scratch/variants/cw23/libmetldpc.so timeout 300 $B > $O/ab_cw23_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$PWD/scratch/variants/cw15/libmetldpc.so timeout 300 $B > $O/ab_cw15_$rep.json 2>>$O/ab.err
done
