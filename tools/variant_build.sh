#!/bin/bash
# Build a variant of librnsw.so with extra -D flags for one source file into ab/<name>.so.
# usage: tools/variant_build.sh <name> <source.cu> [-DFOO=1 ...]
set -e
name=$1; src=$2; shift 2
R=/root/repo
mkdir -p $R/ab/obj_$name
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -I $R/include"
objs=""
for f in $R/paper_2007_12216_b200/build/*.o; do
  b=$(basename $f .o)
  if [ "$b.cu" = "$src" ]; then
    nvcc $FLAGS "$@" -c $R/paper_2007_12216_b200/csrc/$src -o $R/ab/obj_$name/$b.o
    objs="$objs $R/ab/obj_$name/$b.o"
  else
    objs="$objs $f"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $objs -o $R/ab/$name.so -lcudart
rm -rf $R/ab/obj_$name
echo built ab/$name.so
