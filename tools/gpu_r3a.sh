#!/bin/bash
# GPU call: state check after the container re-creation (full suite, smoke, headline) + A/B of the
# L rows staged by the producer warp (batched index loads), parity of the variant, ncu of its (3,1) class
set -x
O=gpurun_out/r3a; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  for m in 32 16; do
    timeout 300 $B --msg-bits $m > $O/ab_base_m${m}_$rep.json 2>>$O/ab.err
    METLDPC_LIB=$V/lst/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_lst_m${m}_$rep.json 2>>$O/ab.err
    METLDPC_LIB=$V/lst19/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_lst19_m${m}_$rep.json 2>>$O/ab.err
  done
done
METLDPC_LIB=$V/lst/libmetldpc.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "c1 or msg16 or refill" > $O/pytest_lst.log 2>&1; echo "rc=$?" >> $O/pytest_lst.log
METLDPC_LIB=$V/lst/libmetldpc.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_ring<0, 3" --launch-skip 1 -c 1 -o $O/ring_lst python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-et --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_default.json 2> $O/bench_default.err
