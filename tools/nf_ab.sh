#!/bin/bash
# RMSNorm folded into the swap-AB GEMVs (just-in-time staging) vs separate rmsnorm launches
for shape in "8b 4 2048" "8b 1 1536" "1b 4 2048" "1b 2 2176"; do
  for t in 0 1; do
    echo -n "nfold=$t :: "; MOA_NORM_FOLD=$t python tools/fwdbench.py $shape 48
  done
done
