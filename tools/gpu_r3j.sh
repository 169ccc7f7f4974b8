#!/bin/bash
# GPU call: refill wave kernels rewritten (lane list + item = lane x 32 VNs): parity, wave cost, thresholds
set -x
O=gpurun_out/r3j; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paths.py -x -q -k "refill or streaming or host or headline or edge" > $O/pytest_refill.log 2>&1; echo "rc=$?" >> $O/pytest_refill.log
timeout 600 python tools/wave_parts.py new 0 $O/wave_parts.jsonl > $O/wp.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for t in 8 4 2 1; do METLDPC_REFILL_MIN=$t timeout 600 $B > $O/bench_t$t.json 2>>$O/err.log; done
