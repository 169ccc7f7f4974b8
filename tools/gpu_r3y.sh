#!/bin/bash
set -x
O=gpurun_out/r3y; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
for w in c1 rand; do for m in 32 16; do
  METLDPC_RING=0 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R $w $m > $O/ring0_${w}_$m.log 2>&1
  METLDPC_RING=0 METLDPC_LIB=$R/scratch/variants/start/libmetldpc.so CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R $w $m > $O/start_ring0_${w}_$m.log 2>&1
  METLDPC_PIPE=0 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R $w $m > $O/pipe0_${w}_$m.log 2>&1
  METLDPC_RING_CORE=0 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R $w $m > $O/core0_${w}_$m.log 2>&1
done; done
