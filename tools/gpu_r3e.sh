#!/bin/bash
# GPU call: L staging with the index loads two stages ahead in rotating registers (A/B vs the old and new base)
set -x
O=gpurun_out/r3e; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for m in 32 16; do
  timeout 300 $B --msg-bits $m > $O/ab_base_m${m}.json 2>>$O/ab.err
  for v in old lst23 lst19p4 lst15p2; do
    METLDPC_LIB=$V/$v/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_${v}_m${m}.json 2>>$O/ab.err
  done
done
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:k_cn_ring<.int.0,..int.3, --launch-skip 1 -c 1"
R="python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e"
METLDPC_LIB=$V/lst19p4/libmetldpc.so timeout 600 $N -o $O/ring_lst19p4 $R > $O/ncu_lst.log 2>&1
METLDPC_LIB=$V/lst19p4/libmetldpc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "c1 or msg16 or refill" > $O/pytest_lst.log 2>&1; echo "rc=$?" >> $O/pytest_lst.log
