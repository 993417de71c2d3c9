#!/bin/bash
# build_variant.sh NAME "EXTRA NVCC FLAGS" -> build/variants/NAME/libdr_raster_b200.so (A/B experiments only)
# FMAD_FILES="raster_bwd ..." compiles those translation units with FMA contraction allowed (-fmad=true).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name; mkdir -p $out
SRCS=$(cd paper_2007_08501_b200/csrc && ls *.cu | sed 's/\.cu$//' | grep -v '^shard_nccl$')
for f in $SRCS; do
  fmad=-fmad=false
  for g in $FMAD_FILES; do [ "$g" = "$f" ] && fmad=-fmad=true; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $fmad -Xcompiler -fPIC -Xptxas -v "$@" \
    -c paper_2007_08501_b200/csrc/$f.cu -o $out/$f.o 2> $out/$f.ptxas.txt &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libdr_raster_b200.so $(for f in $SRCS; do echo $out/$f.o; done) -lcudart
grep -B1 -A3 "Compiling entry function '_ZN3drb6k_fineIfLi8ELi8\|Compiling entry function '_ZN3drb6k_fineIfLi8ELi0" $out/raster_fwd.ptxas.txt | grep -E "registers|spill" | tr '\n' ' '; echo " [$name]"
