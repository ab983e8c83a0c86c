#!/bin/bash
# Round profile capture (run under gpurun from the repo root; never a bench
# number: ncu serialises and replays).  Outputs under gpurun_out/$1/:
#   launches_c3.csv   launch list of a window of one C3 request (bench.py --profile-only)
#   ncu_*.ncu-rep     --set full of the dominant decode / prefill kernels at the
#                     8B / 1B shapes (tools/fwdbench.py ticks)
set -u
R=${1:-prof}
O=gpurun_out/$R
mkdir -p $O
L="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
F="ncu --set full --clock-control none --import-source on -f"
# a window of one C3 request (a whole request is ~6e5 launches): the leaf-phase decode ticks
$L --launch-skip 250000 -c 4000 --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 0 --profile-only > /dev/null 2>&1
$L --launch-skip 900 -c 300 --log-file $O/launches_8b_r4.csv python tools/fwdbench.py 8b 4 2048 16 > /dev/null 2>&1
$L --launch-skip 600 -c 200 --log-file $O/launches_1b_r4.csv python tools/fwdbench.py 1b 4 2048 16 > /dev/null 2>&1
$F -k regex:gemv_tc_kernel --launch-skip 130 -c 3 -o $O/ncu_8b_gemv python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$F -k regex:attention_decode_cluster --launch-skip 40 -c 1 -o $O/ncu_8b_attn_decode python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$F -k regex:lm_head_tc --launch-skip 2 -c 1 -o $O/ncu_8b_lm_head python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$F -k regex:gemm_tc_persistent --launch-skip 2 -c 1 -o $O/ncu_8b_gemm_persistent python tools/fwdbench.py 8b 4 2048 4 > /dev/null 2>&1
$F -k regex:attention_prefill_tc --launch-skip 0 -c 1 -o $O/ncu_8b_attn_prefill_tc python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$F -k regex:gemv_tc_kernel --launch-skip 66 -c 4 -o $O/ncu_1b_gemv python tools/fwdbench.py 1b 4 2048 8 > /dev/null 2>&1
ls -la $O
