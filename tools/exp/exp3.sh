echo "== b2 noise (v4 compensated default)"
timeout 900 python tools/b2_noise.py c4 2>&1 | tail -10
echo "== c4 bench"
timeout 600 python bench.py --config c4 --steps 3 --warmup 1 2>gpurun_out/exp3_c4.err | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['value'], d['kernel_ms_per_step'])"
echo "== gpu tests (compress + typeb)"
timeout 1500 python -m pytest tests/test_gpu_compress.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -5
