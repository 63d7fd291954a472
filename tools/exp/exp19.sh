for c in c3 c4; do timeout 600 python tools/prof_stages.py $c > gpurun_out/stages_$c.txt 2>&1; head -16 gpurun_out/stages_$c.txt; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -s 2>&1 | grep -E "^c[34]|passed|failed" > gpurun_out/fullsize_s.log; cat gpurun_out/fullsize_s.log
mkdir -p gpurun_out/prof
F="--set full --clock-control none --import-source on"
timeout 900 ncu $F -k regex:k_sketch_tagged4 -c 1 -o gpurun_out/prof/c4_sketch4 python tools/one_compress.py c4 1 > gpurun_out/prof/f_c4s.log 2>&1
ncu -i gpurun_out/prof/c4_sketch4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/c4_sketch4_source.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/prof/c4_sketch4_source.csv 45 > gpurun_out/c4_sketch4_lines.txt 2>&1
gzip -f gpurun_out/prof/c4_sketch4_source.csv
ls -la gpurun_out/prof/
rm -f gpurun_out/prof/*.ncu-rep
