#!/bin/bash
# A/B of library variants in paper_2103_05162_b200/ab/*.so with tools/variant_probe.py
# (best-of-5 device time + output digest): tools/ab_probe.sh <tag> C2 [C3 ...]
TAG=$1; shift
mkdir -p gpurun_out
for C in "$@"; do
  for L in paper_2103_05162_b200/ab/*.so; do
    v=$(basename $L .so)
    echo -n "$v " >> gpurun_out/${TAG}_ab.txt
    TCB_LIB_PATH=$PWD/$L timeout 300 python tools/variant_probe.py $C 5 >> gpurun_out/${TAG}_ab.txt 2>> gpurun_out/${TAG}_ab.err
  done
done
cat gpurun_out/${TAG}_ab.txt
