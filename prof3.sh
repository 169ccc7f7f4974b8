for v in P1M3 P1M4 P0M4 P0M3; do
  export METLDPC_LIB=$PWD/build/variants/lib_$v.so
  timeout 300 python -m pytest tests -m gpu -x -q -k "c1 or generic" > gpurun_out/pytest_$v.log 2>&1; echo rc=$? >> gpurun_out/pytest_$v.log
  timeout 300 python bench.py --steps 2 --warmup 1 --frames 64 --iters 20 --distinct 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
unset METLDPC_LIB
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_default3.log 2>&1; echo rc=$? >> gpurun_out/pytest_default3.log
