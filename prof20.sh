export METLDPC_LIB=$PWD/build/variants/lib_PAIR1.so
timeout 900 python -m pytest tests -m gpu -x -q -k "not c3" > gpurun_out/pytest_pair.log 2>&1; echo rc=$? >> gpurun_out/pytest_pair.log
for v in PAIR1 PAIR0 PAIR1 PAIR0; do
  export METLDPC_LIB=$PWD/build/variants/lib_$v.so
  timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups 1 >> gpurun_out/bench_$v.log 2>&1
done
