#!/bin/bash
set -x
O=gpurun_out/r2p; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q -k "refill or streaming or edge or host or headline" > $O/pytest_refill.log 2>&1; echo "rc=$?" >> $O/pytest_refill.log
timeout 900 python tools/wave_cost.py $O/wave_cost.jsonl > $O/wave_cost.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --frames 2048"
for rep in 1 2; do
  timeout 300 $B > $O/ab_cur_$rep.json 2>>$O/ab.err
  METLDPC_LIB=$PWD/scratch/variants/scat_old/libmetldpc.so timeout 300 $B > $O/ab_scatold_$rep.json 2>>$O/ab.err
  METLDPC_REFILL_MIN=4 timeout 300 $B > $O/ab_cur_w4_$rep.json 2>>$O/ab.err
done
