timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_v15.log 2>&1; echo rc=$? >> gpurun_out/pytest_v15.log
timeout 900 python tools/fer_sweep.py --frames 512 --out gpurun_out/r1_fer_sweep.jsonl > gpurun_out/fer.log 2>&1
timeout 900 python tools/batch_sweep.py --out gpurun_out/r1_fig2_sweep.jsonl > gpurun_out/fig2.log 2>&1
timeout 600 python bench.py --family r0.05 --snr 0.076 --iters 150 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
