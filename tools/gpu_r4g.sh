#!/bin/bash
# GPU call: regression test for idle lanes over dirty memory (before / after the fix) + full GPU suite + smoke
set -x
O=gpurun_out/r4g; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
METLDPC_LIB=$PWD/scratch/variants/prefix/libmetldpc.so timeout 600 python -m pytest tests/test_gpu_paths.py -q -k "dirty" > $O/pytest_dirty_prefix.log 2>&1; echo "rc=$?" >> $O/pytest_dirty_prefix.log
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
