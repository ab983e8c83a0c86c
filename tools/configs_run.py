"""One timed request per BASELINE config beyond the headline: C3 (heterogeneous
1B/8B agents, prompt 2k, 512 out), C4 tree vs dense (13 tiny agents), plus
the 8B decode forward rate.  Prints one JSON line per config."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS

PEAKS = ROOT / 'MEASURED_PEAKS.json'
peak = json.load(open(PEAKS))['hbm_gbs'] if PEAKS.exists() else 6544.3
names = sys.argv[1:] or ['C4-tree', 'C4-dense', 'C3']
for name in names:
    cfg = dict(CONFIGS[name])
    t0 = time.time()
    eng, qc = capi.engine_for(cfg)
    setup = time.time() - t0
    eng.run_query(qc, sample=0, resolve=False, detail=False)  # warm-up (graph capture)
    res = []
    for i in range(2 if name != 'C3' else 1):
        r = eng.run_query(qc, sample=i + 1, resolve=False, detail=False)
        res.append(r)
    r = res[-1]
    out = {"config": name, "workload": cfg["workload"], "e2e_ms": r["e2e_ms"], "tokens": r["tokens"],
           "tokens_per_s": r["tokens"] / (r["e2e_ms"] / 1e3), "ticks": r["ticks"], "forwards": r["forwards"],
           "weight_gb": r["weight_bytes"] / 1e9, "weight_stream_gbs": r["weight_bytes"] / 1e9 / (r["e2e_ms"] / 1e3),
           "weight_stream_frac": r["weight_bytes"] / 1e9 / (r["e2e_ms"] / 1e3) / peak, "setup_s": setup,
           "p_requests": len(res)}
    print(json.dumps(out), flush=True)
    eng.close()
