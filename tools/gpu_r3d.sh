#!/bin/bash
# GPU call: L staging with fewer compute warps (deeper ring) and more producer warps
set -x
O=gpurun_out/r3d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for m in 32 16; do
  timeout 300 $B --msg-bits $m > $O/ab_base_m${m}.json 2>>$O/ab.err
  for v in lst19p4 lst15p4 lst11p4 lst15p8; do
    METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_${v}_m${m}.json 2>>$O/ab.err
  done
done
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:k_cn_ring<.int.0,..int.3, --launch-skip 1 -c 1"
R="python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e"
METLDPC_LIB=$V/lst11p4/libmetldpc.so timeout 600 $N -o $O/ring_lst11p4 $R > $O/ncu_lst.log 2>&1
