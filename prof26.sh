timeout 900 python -m pytest tests -m gpu -x -q -k "not c3 and not c4" > gpurun_out/pytest_v16.log 2>&1; echo rc=$? >> gpurun_out/pytest_v16.log
METLDPC_GRAPH=0 timeout 900 python -m pytest tests -m gpu -x -q -k "c1 or invariance" > gpurun_out/pytest_v16_nograph.log 2>&1; echo rc=$? >> gpurun_out/pytest_v16_nograph.log
for gmode in 1 0; do
METLDPC_GRAPH=$gmode timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_graph$gmode.log 2>&1
METLDPC_GRAPH=$gmode timeout 600 python tools/fer_sweep.py --frames 256 --snrs 0.19,0.2 > gpurun_out/fer_graph$gmode.log 2>&1
done
