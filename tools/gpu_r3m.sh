#!/bin/bash
# GPU call: same-box A/B of the blocked lam1 layout against the previous lane-major layout
set -x
O=gpurun_out/r3m; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  METLDPC_REFILL_MIN=2 timeout 600 $B > $O/new_t2_$rep.json 2>>$O/err.log
  METLDPC_REFILL_MIN=2 METLDPC_LIB=$V/oldlam/libmetldpc.so timeout 600 $B > $O/old_t2_$rep.json 2>>$O/err.log
  METLDPC_REFILL_MIN=8 METLDPC_LIB=$V/oldlam/libmetldpc.so timeout 600 $B > $O/old_t8_$rep.json 2>>$O/err.log
done
timeout 600 $B --no-et --frames 256 > $O/new_noet.json 2>>$O/err.log
METLDPC_LIB=$V/oldlam/libmetldpc.so timeout 600 $B --no-et --frames 256 > $O/old_noet.json 2>>$O/err.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
