#!/bin/bash
# ncu launch list of the bench command itself (after it has exited 0 without ncu)
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err || exit 1
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c3_bench.csv > gpurun_out/launches_c3_bench_summary.txt
head -12 gpurun_out/launches_c3_bench_summary.txt; tail -2 gpurun_out/launches_c3_bench_summary.txt
ls -la gpurun_out/launches_c3_bench.csv
