for v in PF0 PF4 PF8; do
  export METLDPC_LIB=$PWD/build/variants/lib_$v.so
  timeout 300 python bench.py --steps 3 --warmup 1 --frames 64 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
done
