#!/bin/bash
# decode-attention A/B (register-staged vs TMA-staged) on decode ticks
for shape in "8b 4 2048" "8b 1 1536" "1b 4 2048" "1b 2 2176"; do
  for t in 0 1; do
    echo -n "tma=$t :: "; MOA_DECODE_TMA=$t python tools/fwdbench.py $shape 48
  done
done
