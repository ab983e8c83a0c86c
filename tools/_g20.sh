timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputests20.log 2>&1; echo tests=$?; grep -E "^FAILED|passed|failed" gpurun_out/gputests20.log | tail -8
grep -E "^E  " gpurun_out/gputests20.log | head -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench20.log 2>&1; echo bench=$?; tail -c 600 gpurun_out/bench20.log
