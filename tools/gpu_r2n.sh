#!/bin/bash
# GPU call: core-class ring compute-warp A/B; headline bench at 4096 frames
set -x
O=gpurun_out/r2n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  timeout 300 $B > $O/ab_cwc15_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$V/cwc11/libmetldpc.so timeout 300 $B > $O/ab_cwc11_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$V/cwc7/libmetldpc.so timeout 300 $B > $O/ab_cwc7_$rep.json 2>>$O/ab.err
  METLDPC_RING_CORE=0 timeout 300 $B > $O/ab_coretile_$rep.json 2>>$O/ab.err
done
timeout 900 python bench.py --no-cpu-baseline > $O/bench_f4096.json 2> $O/bench_f4096.err
timeout 900 python bench.py --no-cpu-baseline --frames 2048 > $O/bench_f2048.json 2> $O/bench_f2048.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring<0, 13" --launch-skip 2 -c 2 -o $O/core python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu_core.log 2>&1
METLDPC_LIB=$V/cwc7/libmetldpc.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring<0, 13" --launch-skip 2 -c 2 -o $O/core7 python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu_core7.log 2>&1
