#!/bin/bash
# GPU call: L staging split over 1/2/4 producer warps (A/B), ncu of base and variants
set -x
O=gpurun_out/r3c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1; do
  for m in 32; do
    timeout 300 $B --msg-bits $m > $O/ab_base_m${m}_$rep.json 2>>$O/ab.err
    for v in lst23 lst19p2 lst19p4; do
      METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_${v}_m${m}_$rep.json 2>>$O/ab.err
    done
  done
done
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:k_cn_ring<.int.0,..int.3, --launch-skip 1 -c 1"
R="python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e"
timeout 600 $N -o $O/ring_base $R > $O/ncu_base.log 2>&1
METLDPC_LIB=$V/lst19p4/libmetldpc.so timeout 600 $N -o $O/ring_lst19p4 $R > $O/ncu_lst.log 2>&1
