for s in "2048 28672 4096" "8192 28672 4096" "8192 6144 4096" "8192 4096 14336" "2048 16384 2048" "1280 3072 2048" "513 16384 2048"; do timeout 120 python tools/gemm_time.py $s; MOA_GEMM_PERSISTENT=0 timeout 120 python tools/gemm_time.py $s 5 | sed 's/^/  tile: /'; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests25.log 2>&1; echo tests=$?; grep -E "^FAILED|passed|failed" gpurun_out/gputests25.log | tail -8
grep -E "^E  " gpurun_out/gputests25.log | head -10
for v in 1 0; do MOA_GEMM_PERSISTENT=$v timeout 300 python tools/fwdbench.py 8b 4 2048 8 | head -1; done
