timeout 300 python tools/exp/strip_gemm.py 2>&1 | head -3
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_compress.py -x -q 2>&1 | tail -2
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('c3', d['value'], d['e2e']['value'], d['roofline']['frac'], d['kernel_ms_per_step'])"
mkdir -p gpurun_out/prof
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:k_gemm3 -c 1 -o gpurun_out/prof/c3_apply_gemm3 python tools/one_compress.py c3 1 > gpurun_out/prof/f_c3b.log 2>&1
python tools/summarize_profiles.py gpurun_out/prof_txt2
rm -f gpurun_out/prof/*.ncu-rep
cat gpurun_out/prof_txt2/c3_apply_gemm3_summary.txt | head -14
