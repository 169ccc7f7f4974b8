#!/bin/bash
# GPU call: blocked lam1 layout (+ degree-1-ordered check classes): full GPU suite, wave parts, headline, A/B
set -x
O=gpurun_out/r3l; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/wave_parts.py blocked 0 $O/wave_parts.jsonl > $O/wp.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for t in 1 2 4; do METLDPC_REFILL_MIN=$t timeout 600 $B > $O/bench_t$t.json 2>>$O/err.log; done
timeout 600 $B --no-et --frames 256 > $O/bench_noet.json 2>>$O/err.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
