#!/bin/bash
# Build libmpgmres_b200.so with extra nvcc defines into tools/variants/<name>.so
# (kernel A/B measurement; select at run time with MPG_LIB_PATH=...).
#   tools/build_variant.sh <name> -DMPG_KB_MINB=4 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/tools/variants
mkdir -p $out /tmp/mpg_var_$name
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -I $root/include -I $root/paper_2109_01232_b200/csrc"
objs=""
for f in $root/paper_2109_01232_b200/csrc/*.cu; do
  o=/tmp/mpg_var_$name/$(basename $f .cu).o
  nvcc $flags "$@" -c $f -o $o &
  objs="$objs $o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/$name.so $objs -lpthread -ldl -lrt
echo $out/$name.so
