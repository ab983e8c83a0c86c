timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests22.log 2>&1; echo tests=$?; grep -E "^FAILED|passed|failed" gpurun_out/gputests22.log | tail -8
grep -E "^E  " gpurun_out/gputests22.log | head -10
for v in 1 0; do MOA_EE_FUSED=$v timeout 600 python bench.py --config C1 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary --concurrency "" --probe-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('EE fused', $v, d['value'], d['ms_per_step'])"; done
