import sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import C2
cfg = dict(C2, out_len=[96, 64, 64])
eng, qc = capi.engine_for(cfg)
r = eng.run_query(qc, sample=0, resolve=False, detail=False)
print('ticks', r['ticks'], 'e2e_ms', r['e2e_ms'])
