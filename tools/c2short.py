"""One short request of a config (default C2, 48 output tokens) for ncu launch
lists:  python tools/c2short.py [out_tokens] [requests] [config]"""
import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
out = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfg = dict(CONFIGS[sys.argv[3] if len(sys.argv) > 3 else 'C2'], out_len=[out, out, out])
eng, qc = capi.engine_for(cfg)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    r = eng.run_query(qc, sample=i, resolve=False, detail=False)
    print('ticks', r['ticks'], 'e2e_ms', round(r['e2e_ms'], 2), flush=True)
