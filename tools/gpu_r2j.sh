#!/bin/bash
# GPU call: refill threshold and batch-size A/B at the headline config; core classes in the ring kernel; parity with it
set -x
O=gpurun_out/r2j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
METLDPC_RING_CORE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "not c3_full and not c4 and not c6" > $O/pytest_ringcore.log 2>&1; echo "rc=$?" >> $O/pytest_ringcore.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for w in 4 8 16 32; do METLDPC_REFILL_MIN=$w timeout 300 $B > $O/wave_$w.json 2>>$O/ab.err; done
timeout 300 $B --frames 256 > $O/frames256.json 2>>$O/ab.err
for rep in 1 2; do
  timeout 300 $B --no-et > $O/core_tile_$rep.json 2>>$O/ab.err
  METLDPC_RING_CORE=1 timeout 300 $B --no-et > $O/core_ring_$rep.json 2>>$O/ab.err
  timeout 300 $B --no-et --msg-bits 16 > $O/core_tile_m16_$rep.json 2>>$O/ab.err
  METLDPC_RING_CORE=1 timeout 300 $B --no-et --msg-bits 16 > $O/core_ring_m16_$rep.json 2>>$O/ab.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_default.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 6 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
METLDPC_RING_CORE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_ringcore.csv python bench.py --steps 1 --warmup 0 --frames 64 --iters 6 --no-et --no-cpu-baseline --no-e2e > /dev/null 2>&1
