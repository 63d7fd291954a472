#!/bin/bash
# Full GPU validation of a build: the -m gpu suite, then the bench lines of every config
# (outputs under gpurun_out/). Run under gpurun.
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; tail -3 gpurun_out/final_gputest.log
timeout 600 python bench.py > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
for c in c4 c2; do timeout 600 python bench.py --config $c > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err; done
timeout 900 python bench.py --config c5 > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err
for c in c3 c4 c2 c5; do python -c "
import json
d = json.load(open('gpurun_out/final_bench_$c.json'))
print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['entry'], d['gpu_launches'])"; done
python -c "
import json
d = json.load(open('gpurun_out/final_bench_ref.json')); print('ref', d['value'], d['impl'], d['cpu_baseline']['cores'])"
python -c "import __graft_entry__ as g; g.smoke()"
