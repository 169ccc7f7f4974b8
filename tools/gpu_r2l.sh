#!/bin/bash
# GPU call: two-CNs-per-warp ring (CPW=2) parity + A/B against CPW=1 and CW=23
set -x
O=gpurun_out/r2l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=$PWD/scratch/variants
METLDPC_LIB=$V/cpw2/libmetldpc.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py tests/test_gpu_paths.py -x -q -k "not c4 and not c6 and not decode_md_host" > $O/pytest_cpw2.log 2>&1; echo "rc=$?" >> $O/pytest_cpw2.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-et --frames 256"
for rep in 1 2; do
  for m in 32 16; do
    timeout 300 $B --msg-bits $m > $O/ab_base_m${m}_$rep.json 2>>$O/ab.err
    METLDPC_LIB=$V/cw23/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_cw23_m${m}_$rep.json 2>>$O/ab.err
    METLDPC_LIB=$V/cpw2/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_cpw2_m${m}_$rep.json 2>>$O/ab.err
    METLDPC_LIB=$V/cpw2w20/libmetldpc.so timeout 300 $B --msg-bits $m > $O/ab_cpw2w20_m${m}_$rep.json 2>>$O/ab.err
  done
done
