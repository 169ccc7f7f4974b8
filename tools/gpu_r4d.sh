#!/bin/bash
set -x
O=gpurun_out/r4d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
for v in nosort nol1tma; do
  METLDPC_LIB=$R/scratch/variants/$v/libmetldpc.so timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/$v.log 2>&1
done
timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/head.log 2>&1
