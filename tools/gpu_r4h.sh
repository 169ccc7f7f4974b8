#!/bin/bash
set -x
O=gpurun_out/r4h; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
METLDPC_LIB=$PWD/scratch/variants/prefix/libmetldpc.so timeout 600 python -m pytest tests/test_gpu_paths.py -q -k "reused" > $O/pytest_prefix.log 2>&1; echo "rc=$?" >> $O/pytest_prefix.log
timeout 600 python -m pytest tests/test_gpu_paths.py -q -k "reused" > $O/pytest_fixed.log 2>&1; echo "rc=$?" >> $O/pytest_fixed.log
