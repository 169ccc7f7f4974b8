#!/bin/bash
set -x
O=gpurun_out/r4c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
KEEP=1 timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/default_keep.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/default_blocking.log 2>&1
METLDPC_GRAPH=0 timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/default_graph0.log 2>&1
METLDPC_LIB=$R/scratch/variants/c_3debbd1/libmetldpc.so timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/c3debbd1.log 2>&1
METLDPC_LIB=$R/scratch/variants/c_6e276c3/libmetldpc.so timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/c6e276c3.log 2>&1
