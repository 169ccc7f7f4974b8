#!/bin/bash
set -x
O=gpurun_out/r4e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
REFILL=0 timeout 300 python tools/alt_debug.py $R c1,rand,c1,rand > $O/norefill.log 2>&1
MSGS=32 timeout 300 python tools/alt_debug.py $R c1,rand,c1,rand,c1 > $O/m32.log 2>&1
MSGS=16 timeout 300 python tools/alt_debug.py $R c1,rand,c1,rand,c1 > $O/m16.log 2>&1
RULES=0 MSGS=16 timeout 300 python tools/alt_debug.py $R c1,c1,c1,c1,c1,c1 > $O/c1x6_m16.log 2>&1
RULES=0 MSGS=32 timeout 300 python tools/alt_debug.py $R c1,c1,c1,c1,c1,c1 > $O/c1x6_m32.log 2>&1
