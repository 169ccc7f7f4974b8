#!/bin/bash
set -x
O=gpurun_out/r3z2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
for w in c1 rand c1,rand; do
  METLDPC_RING=0 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R $w > $O/ring0_$w.log 2>&1
done
METLDPC_RING=0 CUDA_LAUNCH_BLOCKING=1 METLDPC_GRAPH=0 timeout 300 python tools/alt_debug.py $R c1,rand > $O/ring0_graph0.log 2>&1
