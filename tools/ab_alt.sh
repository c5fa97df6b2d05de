#!/bin/bash
# A/B of step-kernel build variants at cfg2 (solve times interleaved, phase timelines, bitwise hashes)
# usage: tools/ab_alt.sh variant1 variant2 ...   ("default" = the in-tree library)
out=gpurun_out/ab_alt.log
: > $out
lib() { [ "$1" = default ] && echo "" || echo "tools/variants/$1.so"; }
for v in "$@"; do
  MPG_LIB_PATH=$(lib $v) python tools/hash_solve.py laplace3d 60 ir >> $out 2>&1
  MPG_LIB_PATH=$(lib $v) python tools/hash_solve.py laplace3d 40 fp64 >> $out 2>&1
done
for r in 1 2; do
  for v in "$@"; do
    echo "== $v" >> $out
    MPG_LIB_PATH=$(lib $v) python tools/solve_time.py --reps 3 >> $out 2>&1
  done
done
for v in mt mtalt; do
  [ -f tools/variants/$v.so ] || continue
  echo "== phases $v" >> $out
  MPG_LIB_PATH=tools/variants/$v.so python tools/mega_phases.py 150 >> $out 2>&1
done
cat $out
