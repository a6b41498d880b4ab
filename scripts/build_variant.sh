#!/bin/bash
# Build an experimental libomniseg.so with extra -D flags into paper_2305_14566_b200/lib/<name>/;
# select it at run time with OMNISEG_LIB=<path>.  Usage: scripts/build_variant.sh NAME -DFOO ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/paper_2305_14566_b200/lib/$name
mkdir -p $out
for s in omniseg conv_tc kernels; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -I$root/include "$@" -c $root/paper_2305_14566_b200/csrc/$s.cu -o $out/$s.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libomniseg.so $out/*.o -ldl
echo $out/libomniseg.so
