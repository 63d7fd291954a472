#!/bin/bash
# Launch lists and ncu --set full captures of the bench's dominant kernels,
# into gpurun_out/prof/. Run under gpurun, after the same commands exited 0
# without ncu. Summarise here with tools/summarize_profiles.py into profiles/.
#   tools/profile_round.sh [c2] [c3] [c5]      (default: c2)
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
CFGS=${*:-c2}
M="--metrics gpu__time_duration.sum --clock-control none --csv"
F="--set full --clock-control none --import-source on"
for c in $CFGS; do
  python tools/one_compress.py $c 1 > /dev/null 2>&1 || { echo "plain run $c failed"; exit 1; }
done
for c in $CFGS; do
  case $c in
    c2)
      # the bench command itself (launch list), then one compression per capture
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/b_c2.log 2>&1 || { echo "bench c2 failed"; exit 1; }
      ncu $M -c 400 --log-file $OUT/launches_c2_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/l_c2b.log 2>&1
      ncu $M --log-file $OUT/launches_c2.csv python tools/one_compress.py c2 2 > $OUT/l_c2.log 2>&1
      ncu $F -k regex:k_sketch_tagged4 -s 1 -c 1 -o $OUT/c2_sketch4 python tools/one_compress.py c2 2 > $OUT/f_c2s.log 2>&1
      ncu $F -k regex:k_coupling_nf_small -s 1 -c 1 -o $OUT/c2_cnf python tools/one_compress.py c2 2 > $OUT/f_c2c.log 2>&1
      ;;
    c3)
      ncu $M --log-file $OUT/launches_c3.csv python tools/one_compress.py c3 1 > $OUT/l_c3.log 2>&1
      # the staged apply: first k_gen_strip and first k_gemm3 launch (one full strip each);
      # a later k_gemm3 launch is a block-nullification product
      ncu $F -k regex:k_gen_strip -c 1 -o $OUT/c3_gen_strip python tools/one_compress.py c3 1 > $OUT/f_c3a.log 2>&1
      ncu $F -k regex:k_gemm3 -c 1 -o $OUT/c3_apply_gemm3 python tools/one_compress.py c3 1 > $OUT/f_c3b.log 2>&1
      ncu $F -k regex:k_gemm3 -s 10 -c 1 -o $OUT/c3_gemm3 python tools/one_compress.py c3 1 > $OUT/f_c3g.log 2>&1
      ;;
    c4)
      ncu $F -k regex:k_sketch_tagged4 -c 1 -o $OUT/c4_sketch4 python tools/one_compress.py c4 1 > $OUT/f_c4s.log 2>&1
      ;;
    c5)
      ncu $M --log-file $OUT/launches_c5.csv python tools/one_compress.py c5 1 > $OUT/l_c5.log 2>&1
      ncu $F -k regex:k_sketch_tagged4 -c 1 -o $OUT/c5_sketch4 python tools/one_compress.py c5 1 > $OUT/f_c5s.log 2>&1
      ncu $F -k regex:k_coupling3 -c 1 -o $OUT/c5_coupling3 python tools/one_compress.py c5 1 > $OUT/f_c5c.log 2>&1
      ;;
  esac
done
# summarise on the box and drop the reports (several full captures exceed the
# 64 MiB that gpurun copies back)
python tools/summarize_profiles.py gpurun_out/prof_txt
rm -f $OUT/*.ncu-rep
echo done
