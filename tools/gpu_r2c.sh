#!/bin/bash
# GPU call: k_cn_ring parity + A/B vs k_cn_pipe (fp32 and 16-bit messages)
set -x
O=gpurun_out/r2c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
METLDPC_RING=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q > $O/pytest_ring.log 2>&1; echo "rc=$?" >> $O/pytest_ring.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for rep in 1 2; do
  timeout 300 $B > $O/ab_pipe_$rep.json 2>>$O/ab.err
  METLDPC_RING=1 timeout 300 $B > $O/ab_ring_$rep.json 2>>$O/ab.err
  timeout 300 $B --msg-bits 16 > $O/ab_pipe_m16_$rep.json 2>>$O/ab.err
  METLDPC_RING=1 timeout 300 $B --msg-bits 16 > $O/ab_ring_m16_$rep.json 2>>$O/ab.err
done
METLDPC_RING=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_(ring|tile)" --launch-skip 3 -c 3 -o $O/ring_m16 python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-cpu-baseline --no-e2e --msg-bits 16 > $O/ncu_ring.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn_(pipe|tile)" --launch-skip 3 -c 3 -o $O/pipe_m16 python bench.py --steps 1 --warmup 0 --frames 64 --iters 8 --no-cpu-baseline --no-e2e --msg-bits 16 > $O/ncu_pipe.log 2>&1
