import sys, os
sys.path.insert(0, '/root/repo')
os.environ['MOA_HOST_PROFILE'] = '1'
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import C1, C0
for cfg in (C0, C1):
    eng, qc = capi.engine_for(cfg)
    for i in range(4):
        r = eng.run_query(qc, sample=i, resolve=False, detail=False)
        print(cfg['name'], 'e2e_ms', round(r['e2e_ms'], 2), 'wall_ms', round(r['wall_ms'], 2), 'ticks', r['ticks'], flush=True)
    eng.close()
