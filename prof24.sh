python - <<'PY' > gpurun_out/l2attr.txt
import ctypes, torch
p=torch.cuda.get_device_properties(0)
print(p)
PY
nvidia-smi -q | grep -i -A3 "l2\|persist" | head -20 >> gpurun_out/l2attr.txt
for cfg in "1 1" "1 0" "4 1" "4 0"; do set -- $cfg
METLDPC_L2PERSIST=$2 timeout 300 python bench.py --steps 3 --warmup 1 --frames 256 --iters 30 --distinct 8 --no-e2e --no-cpu-baseline --groups $1 > gpurun_out/bench_l2_$1_$2.log 2>&1
done
