#!/bin/bash
# GPU call: streaming pass tail in one launch (finish + latch by the last block): parity + same-box A/B
set -x
O=gpurun_out/r3t; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py tests/test_gpu_msg16.py -x -q -k "refill or streaming or host or headline or edge or invariance" > $O/pytest_refill.log 2>&1; echo "rc=$?" >> $O/pytest_refill.log
V=$PWD/scratch/variants
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2 3; do
  timeout 600 $B > $O/new_$rep.json 2>>$O/err.log
  METLDPC_LIB=$V/seplatch/libmetldpc.so timeout 600 $B > $O/old_$rep.json 2>>$O/err.log
done
