#!/bin/bash
# A/B of the weight-stream run-ahead (MOA_PF_MB window, evict-first, wrap) on decode ticks
for shape in "8b 4 2048" "8b 1 1536" "1b 4 2048" "1b 2 2176"; do
  for cfg in "0 0 0" "0 1 0" "32 1 0" "64 1 0" "96 1 0" "64 0 0" "64 1 1"; do
    set -- $cfg
    echo -n "pf=$1 ef=$2 wrap=$3 :: "
    MOA_PF_MB=$1 MOA_EVICT_FIRST=$2 MOA_PF_WRAP=$3 python tools/fwdbench.py $shape 48
  done
done
