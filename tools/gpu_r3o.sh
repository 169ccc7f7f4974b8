#!/bin/bash
# GPU call: pair rows (r, L, lam_a, 64-bit accumulator words): full GPU suite, smoke, same-box A/B vs the lane-order rows
set -x
O=gpurun_out/r3o; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 600 $B --no-et --frames 256 > $O/new_noet_$rep.json 2>>$O/err.log
  METLDPC_LIB=$V/prepair/libmetldpc.so timeout 600 $B --no-et --frames 256 > $O/old_noet_$rep.json 2>>$O/err.log
  timeout 600 $B --no-et --frames 256 --msg-bits 16 > $O/new_noet_m16_$rep.json 2>>$O/err.log
  METLDPC_LIB=$V/prepair/libmetldpc.so timeout 600 $B --no-et --frames 256 --msg-bits 16 > $O/old_noet_m16_$rep.json 2>>$O/err.log
  timeout 600 $B > $O/new_$rep.json 2>>$O/err.log
  METLDPC_LIB=$V/prepair/libmetldpc.so timeout 600 $B > $O/old_$rep.json 2>>$O/err.log
done
