timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_compress.py tests/test_distributed.py -x -q 2>&1 | tail -3
for c in c3 c4; do timeout 600 python tools/prof_stages.py $c > gpurun_out/stages_$c.txt 2>&1; head -14 gpurun_out/stages_$c.txt; done
