#!/bin/bash
set -x
O=gpurun_out/r4a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
for c in 3debbd1 6e276c3 59439fa; do
  METLDPC_RING=0 METLDPC_LIB=$R/scratch/variants/c_$c/libmetldpc.so timeout 300 python tools/alt_debug.py $R c1,rand > $O/ring0_$c.log 2>&1
done
METLDPC_RING=0 timeout 300 python tools/alt_debug.py $R rand,c1 > $O/ring0_head_randfirst.log 2>&1
