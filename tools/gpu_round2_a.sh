#!/bin/bash
# GPU call: parity suite, smoke, a short bench, compute-sanitizer on C1
set -x
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a/smoke.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_c1.py > gpurun_out/r2a/sanitize_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/sanitize_$t.log
done
METLDPC_GRAPH=0 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_c1.py > gpurun_out/r2a/sanitize_racecheck_graph0.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/sanitize_racecheck_graph0.log
