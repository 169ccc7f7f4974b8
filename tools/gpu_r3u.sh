#!/bin/bash
# GPU call: core-class compute warps 15 (base) vs 12
set -x
O=gpurun_out/r3u; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  timeout 300 $B > $O/ab_base_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$V/cwc12/libmetldpc.so timeout 300 $B > $O/ab_cwc12_$rep.json 2>>$O/ab.err
done
