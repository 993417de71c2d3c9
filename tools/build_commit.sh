#!/bin/bash
# build_commit.sh COMMIT NAME -> build/variants/NAME/libdr_raster_b200.so built from COMMIT's sources (A/B only)
set -e
cd "$(dirname "$0")/.."
commit=$1; name=$2
wt=/tmp/wt_$name
rm -rf $wt; git worktree add -f $wt $commit >/dev/null 2>&1
out=$PWD/build/variants/$name; mkdir -p $out
SRCS=$(cd $wt/paper_2007_08501_b200/csrc && ls *.cu | sed 's/\.cu$//' | grep -v '^shard_nccl$')
for f in $SRCS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -Xptxas -v -I$wt/include \
    -c $wt/paper_2007_08501_b200/csrc/$f.cu -o $out/$f.o 2> $out/$f.ptxas.txt &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libdr_raster_b200.so $(for f in $SRCS; do echo $out/$f.o; done) -lcudart
git worktree remove --force $wt
echo "built $name from $commit"
