for stg in 1 0; do
UBLR_APPLY_STAGED=$stg timeout 300 python tools/apply_variants.py 2>&1 | tail -11
done
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline 2>gpurun_out/exp7.err | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c3', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['entry'], d['gpu_launches']); print(d['kernel_ms_per_step'])"
timeout 600 python bench.py --config c4 --steps 3 --warmup 1 --no-cpu-baseline 2>>gpurun_out/exp7.err | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c4', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['entry']); print(d['kernel_ms_per_step'])"
