#!/bin/bash
set -x
O=gpurun_out/r4f; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
R=$PWD
RULES=0 MSGS=16 timeout 300 python tools/alt_debug.py $R c1,c1,c1,c1,c1,c1 > $O/c1x6_m16.log 2>&1
timeout 300 python tools/alt_debug.py $R c1,rand,c1,rand > $O/mix.log 2>&1
METLDPC_RING=0 timeout 300 python tools/alt_debug.py $R c1,rand,c1 > $O/ring0.log 2>&1
timeout 900 python -m pytest tests/test_gpu_paths.py -x -q -k "alternative" > $O/pytest_alt.log 2>&1; echo rc=$? >> $O/pytest_alt.log
