#!/bin/bash
# Builds A/B variants of the library into paper_2103_05162_b200/ab/ (git-ignored,
# travels to the GPU box): tools/build_variants.sh name "-DMACRO=.." [name "..."]...
set -e
cd "$(dirname "$0")/../paper_2103_05162_b200/csrc"
mkdir -p ../ab
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -j16 EXTRA="$flags" OBJDIR=build_ab_$name OUT=../ab/libtreeclust_b200_$name.so >/dev/null 2>&1 \
    || { echo "build $name failed"; exit 1; }
  rm -rf build_ab_$name  # objects are not needed once linked (keeps the gpurun snapshot small)
  echo "built ab/libtreeclust_b200_$name.so ($flags)"
done
