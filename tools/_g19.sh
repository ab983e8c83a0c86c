timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests19.log 2>&1; echo tests=$?; grep -E "^FAILED|passed|failed" gpurun_out/gputests19.log | tail -8
grep -E "^E  " gpurun_out/gputests19.log | head -10
for a in "8b 4 2048" "8b 1 1200" "1b 4 2048" "1b 2 1200"; do timeout 300 python tools/fwdbench.py $a 48; done 2>&1 | tee gpurun_out/fwd19.log
timeout 400 python tools/chaindec.py 8b 4 2048 16 > gpurun_out/chain19_8b4.log 2>&1; grep -v records gpurun_out/chain19_8b4.log | tail -16
