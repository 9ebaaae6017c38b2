#!/bin/bash
# build an alternative libfsqr.so with extra nvcc defines for one source, for A/B measurements:
#   tools/build_variant.sh <name> <source.cu> -DMACRO=VALUE ...   ->  build_var/<name>/libfsqr.so
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
python -c "import paper_2601_02826_b200._build as b; b.build()"
out=build_var/$name; mkdir -p $out
objs=""
for o in paper_2601_02826_b200/build/*.o; do
  b=$(basename $o .o)
  if [ "$b.cu" = "$src" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" \
      -c paper_2601_02826_b200/csrc/$src -o $out/$b.o
    objs="$objs $out/$b.o"
  else
    objs="$objs $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o $out/libfsqr.so $objs
echo $out/libfsqr.so
