#!/bin/bash
# ncu --set full captures of the hot kernels at the 8B / 1B shapes (one kernel
# each, read back here with ncu -i ... --page raw --csv) + a launch list of
# 8B decode ticks.  Never a number for the bench: ncu serialises and replays.
set -x
O=gpurun_out/prof_r2
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:gemv_tc_kernel --launch-skip 130 -c 1 -o $O/ncu_8b_gemv_gate_up -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:gemv_tc_kernel --launch-skip 131 -c 1 -o $O/ncu_8b_gemv_down -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:gemv_tc_kernel --launch-skip 128 -c 1 -o $O/ncu_8b_gemv_qkv -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:attention_decode_tma --launch-skip 40 -c 1 -o $O/ncu_8b_attn_decode -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:lm_head_tc --launch-skip 2 -c 1 -o $O/ncu_8b_lm_head -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:gemm_tc_kernel --launch-skip 2 -c 1 -o $O/ncu_8b_gemm_gate_up -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:attention_prefill_mma --launch-skip 0 -c 1 -o $O/ncu_8b_attn_prefill -f python tools/fwdbench.py 8b 4 2048 8 > /dev/null 2>&1
$NCU -k regex:gemv_tc_kernel --launch-skip 66 -c 1 -o $O/ncu_1b_gemv_gate_up -f python tools/fwdbench.py 1b 4 2048 8 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 900 -c 330 --csv --log-file $O/launches_8b_r4.csv python tools/fwdbench.py 8b 4 2048 16 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 900 -c 200 --csv --log-file $O/launches_1b_r4.csv python tools/fwdbench.py 1b 4 2048 16 > /dev/null 2>&1
ls -la $O
