#!/bin/bash
# Launch lists (one compression after warm-up) and ncu --set full captures of
# each config's dominant kernel, into gpurun_out/prof/. Run under gpurun, after
# the same commands exited 0 without ncu. Summarise here with
# tools/launch_summary.py and tools/ncu_summary.py into profiles/.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
M="--metrics gpu__time_duration.sum --clock-control none --csv"
for c in c2 c3 c5; do
  python tools/one_compress.py $c 1 > /dev/null 2>&1 || { echo "plain run $c failed"; exit 1; }
done
ncu $M --log-file $OUT/launches_c2.csv python tools/one_compress.py c2 2 > $OUT/l_c2.log 2>&1
ncu $M --log-file $OUT/launches_c3.csv python tools/one_compress.py c3 1 > $OUT/l_c3.log 2>&1
ncu $M --log-file $OUT/launches_c5.csv python tools/one_compress.py c5 1 > $OUT/l_c5.log 2>&1
F="--set full --clock-control none --import-source on"
ncu $F -k regex:k_sketch_tagged3 -s 1 -c 1 -o $OUT/c2_sketch3 python tools/one_compress.py c2 2 > $OUT/f_c2.log 2>&1
ncu $F -k regex:k_apply3 -c 1 -o $OUT/c3_apply3 python tools/one_compress.py c3 1 > $OUT/f_c3.log 2>&1
ncu $F -k regex:k_sketch_tagged3 -c 1 -o $OUT/c5_sketch3 python tools/one_compress.py c5 1 > $OUT/f_c5s.log 2>&1
ncu $F -k regex:k_coupling3 -c 1 -o $OUT/c5_coupling3 python tools/one_compress.py c5 1 > $OUT/f_c5c.log 2>&1
echo done
