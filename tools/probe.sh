#!/bin/bash
# Work counters of the instrumented build (make -C paper_2103_05162_b200/csrc probe)
# for the given configs: tools/probe.sh C2 [C3fd ...]
mkdir -p gpurun_out
TCB_LIB_PATH=$PWD/paper_2103_05162_b200/libtreeclust_b200_probe.so \
  python tools/configs.py "$@" 2>&1 | grep -E "^\[probe\]|config" | tail -n 20
