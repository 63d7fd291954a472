timeout 600 python tools/exp/strip_gemm.py 2>&1 | head -4
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/s4_bench_c3_c.json 2> gpurun_out/s4_bench_c3_c.err
python -c "
import json
d = json.load(open('gpurun_out/s4_bench_c3_c.json'))
print('c3', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['entry'], d['gpu_launches']); print(d['kernel_ms_per_step'])"
