#!/bin/bash
# GPU call: cost of the lane-list wave kernels (each launched twice in a variant) + tiny-kernel node cost
set -x
O=gpurun_out/r3k; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
for rep in 1 2; do
timeout 600 python tools/wave_parts.py new 0 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/nwrep1/libmetldpc.so timeout 600 python tools/wave_parts.py finalize 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/nwrep2/libmetldpc.so timeout 600 python tools/wave_parts.py scatter 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/nwrep8/libmetldpc.so timeout 600 python tools/wave_parts.py activate 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
done
