#!/bin/bash
# GPU call: msg16 parity, LTMA variant A/B on C3 (fp32 / 16-bit messages), sanitizer isolation
set -x
O=gpurun_out/r2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_msg16.py -x -q > $O/pytest_msg16.log 2>&1; echo "rc=$?" >> $O/pytest_msg16.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
LT=$PWD/scratch/variants/ltma/libmetldpc.so
for rep in 1 2; do
  timeout 300 $B > $O/ab_base_$rep.json 2>>$O/ab.err
  timeout 300 $B --msg-bits 16 > $O/ab_m16_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$LT timeout 300 $B > $O/ab_ltma_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$LT timeout 300 $B --msg-bits 16 > $O/ab_ltma_m16_$rep.json 2>>$O/ab.err
done
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9"
timeout 600 $SAN --tool memcheck python tools/sanitize_c1.py > $O/memcheck_default.log 2>&1; echo "rc=$?" >> $O/memcheck_default.log
METLDPC_PDL=0 timeout 600 $SAN --tool memcheck python tools/sanitize_c1.py > $O/memcheck_pdl0.log 2>&1; echo "rc=$?" >> $O/memcheck_pdl0.log
METLDPC_GRAPH=0 timeout 600 $SAN --tool memcheck python tools/sanitize_c1.py > $O/memcheck_graph0.log 2>&1; echo "rc=$?" >> $O/memcheck_graph0.log
METLDPC_PDL=0 timeout 600 $SAN --tool synccheck python tools/sanitize_c1.py > $O/synccheck_pdl0.log 2>&1; echo "rc=$?" >> $O/synccheck_pdl0.log
METLDPC_GRAPH=0 timeout 600 $SAN --tool synccheck python tools/sanitize_c1.py > $O/synccheck_graph0.log 2>&1; echo "rc=$?" >> $O/synccheck_graph0.log
