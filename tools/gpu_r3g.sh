#!/bin/bash
# GPU call: groups in flight for the streaming headline (K = 1 / 2 / 3), refill threshold at K = 2
set -x
O=gpurun_out/r3g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  for k in 1 2 3; do
    timeout 600 $B --groups $k > $O/k${k}_$rep.json 2>>$O/err.log
  done
done
for t in 4 16; do METLDPC_REFILL_MIN=$t timeout 600 $B --groups 2 > $O/k2_t$t.json 2>>$O/err.log; done
timeout 600 $B --groups 2 --msg-bits 16 > $O/k2_m16.json 2>>$O/err.log
timeout 600 $B --groups 1 --msg-bits 16 > $O/k1_m16.json 2>>$O/err.log
