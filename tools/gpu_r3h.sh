#!/bin/bash
# GPU call: ring compute warps 23 (80 regs) vs 24 / 27 (72 regs)
set -x
O=gpurun_out/r3h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  timeout 300 $B > $O/ab_base_$rep.json 2>>$O/ab.err
  for v in cw24 cw27; do METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B > $O/ab_${v}_$rep.json 2>>$O/ab.err; done
done
