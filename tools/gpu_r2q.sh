#!/bin/bash
set -x
O=gpurun_out/r2q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
METLDPC_LIB=$V/half16/libmetldpc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py tests/test_gpu_paths.py -x -q -k "c1 or generic or r01de or msg16 or headline" > $O/pytest_half16.log 2>&1; echo "rc=$?" >> $O/pytest_half16.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  for m in 32 16; do
  timeout 300 $B --msg-bits $m > $O/ab_base_m${m}_$rep.json 2>>$O/ab.err
  for v in half16 half20 half; do
    METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_${v}_m${m}_$rep.json 2>>$O/ab.err
  done
  done
done
METLDPC_LIB=$V/half16/libmetldpc.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring<0, 13" --launch-skip 2 -c 2 -o $O/core_half16 python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
