"""Throughput of concurrent requests (continuous batching) per config:
python tools/batchrun.py C1 1 2 4 8"""
import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
name = sys.argv[1]
for b in [int(x) for x in sys.argv[2:]]:
    cfg = dict(CONFIGS[name])
    eng, qc = capi.engine_for(cfg, concurrency=b)
    eng.run_batch(qc, list(range(b)), resolve=False, detail=False)
    rs = eng.run_batch(qc, [b + i for i in range(b)], resolve=False, detail=False)
    batch_ms = max(r["e2e_ms"] for r in rs)
    toks = sum(r["tokens"] for r in rs)
    lat = sorted(r["e2e_ms"] for r in rs)
    print(f"{name} concurrency {b}: {toks / (batch_ms / 1e3):.0f} tokens/s, batch {batch_ms:.2f} ms, "
          f"per-request p50 {lat[len(lat) // 2]:.2f} ms, ticks {rs[0]['ticks']}", flush=True)
    eng.close()
