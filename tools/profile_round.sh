#!/bin/bash
# Round profile capture (run under gpurun from the repo root): launch lists of
# the headline (C1) and the 1B decode (C2) workloads, and full ncu sections of
# the dominant kernels.  Outputs under gpurun_out/$1/.
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
NCU="ncu --clock-control none"
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 1 --profile-only > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum --csv --log-file $O/launches_c2.csv python tools/c2short.py 48 1 C2 > /dev/null 2>&1
# full sections: C1 decode-tick fused QKV+attention and LM head; 1B decode GEMVs, LM head, attention
$NCU --set full --import-source on -k regex:qkv_attention -s 300 -c 1 -o $O/ncu_c1_qkv_attention python tools/c2short.py 16 1 C1 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:gemv_kernel -s 300 -c 3 -o $O/ncu_c1_gemv python tools/c2short.py 16 1 C1 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:lm_head_tc -s 10 -c 1 -o $O/ncu_c1_lm_head python tools/c2short.py 16 1 C1 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:gemv_tc -s 300 -c 4 -o $O/ncu_c2_gemv_tc python tools/c2short.py 16 1 C2 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:lm_head_tc -s 10 -c 1 -o $O/ncu_c2_lm_head python tools/c2short.py 16 1 C2 > /dev/null 2>&1
$NCU --set full --import-source on -k regex:attention_gqa -s 300 -c 1 -o $O/ncu_c2_attention python tools/c2short.py 16 1 C2 > /dev/null 2>&1
ls -la $O
