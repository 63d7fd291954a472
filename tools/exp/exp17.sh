timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputest4.log 2>&1; tail -3 gpurun_out/s4_gputest4.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for c in c4 c2; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c3 c4 c2 c5; do python -c "
import json
d = json.load(open('gpurun_out/bench_$c.json'))
print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['entry'], d['gpu_launches'], d.get('cpu_baseline', {}) and d['cpu_baseline'].get('value'))"; done
