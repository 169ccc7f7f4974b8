#!/bin/bash
# GPU call: parity of the A/B alternatives (per-warp pipeline, register-only tiles) on the pair rows / blocked lam1
set -x
O=gpurun_out/r3w; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
K="c1 or degree1 or generic or invariance or refill or msg16 or pair_acc"
METLDPC_RING=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "$K" > $O/pytest_ring0.log 2>&1; echo "rc=$?" >> $O/pytest_ring0.log
METLDPC_RING_CORE=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "$K" > $O/pytest_core0.log 2>&1; echo "rc=$?" >> $O/pytest_core0.log
METLDPC_PIPE=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_msg16.py -x -q -k "$K" > $O/pytest_pipe0.log 2>&1; echo "rc=$?" >> $O/pytest_pipe0.log
