#!/bin/bash
# GPU call: phi table with 4 copies (2-way bank conflicts, half the table, deeper ring) vs 8 copies
set -x
O=gpurun_out/r3n; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  timeout 300 $B > $O/ab_base_$rep.json 2>>$O/ab.err
  for v in cp4 cp4s8; do METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B > $O/ab_${v}_$rep.json 2>>$O/ab.err; done
done
METLDPC_LIB=$V/cp4/libmetldpc.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1" > $O/pytest_cp4.log 2>&1; echo "rc=$?" >> $O/pytest_cp4.log
