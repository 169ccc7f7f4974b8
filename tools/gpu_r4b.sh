#!/bin/bash
set -x
O=gpurun_out/r4b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
METLDPC_RING=0 METLDPC_PDL=0 timeout 300 python tools/alt_debug.py $R c1,rand > $O/ring0_pdl0.log 2>&1
METLDPC_RING=0 METLDPC_L2PERSIST=0 timeout 300 python tools/alt_debug.py $R c1,rand > $O/ring0_l2p0.log 2>&1
METLDPC_RING=0 timeout 300 python tools/alt_debug.py $R rand,rand > $O/ring0_randrand.log 2>&1
METLDPC_RING=0 timeout 300 python tools/alt_debug.py $R c1,c1 > $O/ring0_c1c1.log 2>&1
timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/default_c1randc1.log 2>&1
