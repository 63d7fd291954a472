timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "sketch" 2>&1 | tail -3
for c in c4 c5; do
timeout 240 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>>gpurun_out/exp21.err | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', d['value'], {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items() if 'sketch' in k}, d['gpu_launches'])"
done
