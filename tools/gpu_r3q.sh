#!/bin/bash
# GPU call: cost of one WHILE-body iteration (group graph with 2 passes per body) + the new hi-lane message tests
set -x
O=gpurun_out/r3q; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "messages_every_iteration" > $O/pytest_msgs.log 2>&1; echo "rc=$?" >> $O/pytest_msgs.log
V=$PWD/scratch/variants
for rep in 1 2; do
  timeout 600 python tools/pass_cost.py base $O/pass_cost.jsonl >> $O/log.txt 2>&1
  METLDPC_LIB=$V/unroll2/libmetldpc.so timeout 600 python tools/pass_cost.py unroll2 $O/pass_cost.jsonl >> $O/log.txt 2>&1
done
