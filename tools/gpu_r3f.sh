#!/bin/bash
# GPU call: timing probe of 8-byte lane-pair accesses (LDG/LDS/STG/RED .64) in the ring kernel (wrong layout, timing only)
set -x
O=gpurun_out/r3f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  timeout 300 $B > $O/ab_base_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$V/probe/libmetldpc.so timeout 300 $B > $O/ab_probe_$rep.json 2>>$O/ab.err
done
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:k_cn_ring<.int.0,..int.3, --launch-skip 1 -c 1"
R="python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e"
METLDPC_LIB=$V/probe/libmetldpc.so timeout 600 $N -o $O/ring_probe $R > $O/ncu_probe.log 2>&1
