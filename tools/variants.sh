#!/bin/bash
# A/B kernel variants on the GPU box: tools/variants.sh <tag> <config> <VAR> <v1> [v2 ...]
# One process per value (the variables are read once per process).
TAG=$1; CFG=$2; VAR=$3; shift 3
mkdir -p gpurun_out
for v in "$@"; do
  env "$VAR=$v" timeout 300 python tools/variant_probe.py "$CFG" 5 >> gpurun_out/${TAG}_variants.jsonl 2>> gpurun_out/${TAG}_variants.err
done
cat gpurun_out/${TAG}_variants.jsonl
