#!/bin/bash
# GPU call: cost of the refill-wave parts (each idempotent wave kernel launched twice in a variant)
set -x
O=gpurun_out/r3i; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
for rep in 1 2; do
timeout 600 python tools/wave_parts.py base 0 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/wrep1/libmetldpc.so timeout 600 python tools/wave_parts.py finalize 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/wrep2/libmetldpc.so timeout 600 python tools/wave_parts.py scatter 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
METLDPC_LIB=$V/wrep4/libmetldpc.so timeout 600 python tools/wave_parts.py synd 1 $O/wave_parts.jsonl >> $O/log.txt 2>&1
done
