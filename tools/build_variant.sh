#!/bin/bash
# Build an experimental libpoly_b200 variant with extra -D flags into tools/lib12/<name>.so
# (git-ignored; selected at run time with POLY_B200_LIB=...).  Usage: build_variant.sh name -DX=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
out=tools/lib12/$name; mkdir -p $out
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $*"
for s in $(python3 -c "import sys; sys.path.insert(0, 'paper_1609_01882_b200'); import build; print(' '.join(x[:-3] for x in build.SOURCES))"); do
  /usr/local/cuda/bin/nvcc $F -c paper_1609_01882_b200/csrc/$s.cu -o $out/$s.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $out/*.o -o tools/lib12/$name.so -lcudart
echo tools/lib12/$name.so
