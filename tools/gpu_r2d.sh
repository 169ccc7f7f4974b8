#!/bin/bash
# GPU call: full parity suite + smoke on the ring default, bench lines (fp32 / 16-bit / LUT), sanitizers (host loop)
set -x
O=gpurun_out/r2d; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_exact.json 2> $O/bench_c3_exact.err
timeout 600 python bench.py --msg-bits 16 > $O/bench_c3_exact_m16.json 2> $O/bench_c3_exact_m16.err
timeout 600 python bench.py --rule lut --msg-bits 16 --no-cpu-baseline > $O/bench_c3_lut_m16.json 2> $O/bench_c3_lut_m16.err
SAN="compute-sanitizer --print-limit 20 --error-exitcode 9 --num-cuda-barriers 40000"
for t in memcheck racecheck synccheck; do
  METLDPC_GRAPH=0 timeout 900 $SAN --tool $t python tools/sanitize_c1.py > $O/sanitize_${t}_graph0.log 2>&1; echo "rc=$?" >> $O/sanitize_${t}_graph0.log
done
timeout 900 $SAN --tool racecheck python tools/sanitize_c1.py > $O/sanitize_racecheck_graph.log 2>&1; echo "rc=$?" >> $O/sanitize_racecheck_graph.log
