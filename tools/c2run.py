import json, time, sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import C2, C3
for cfg in (C2,):
    t0 = time.time()
    eng, qc = capi.engine_for(cfg)
    t1 = time.time()
    for i in range(2):
        r = eng.run_query(qc, sample=i, resolve=True, detail=True)
        print(cfg['name'], 'setup_s', round(t1-t0,1), 'e2e_ms', round(r['e2e_ms'],1), 'ticks', r['ticks'], 'tokens', r['tokens'], 'host_ms', round(r['host_ms'],1), 'tok/s', round(r['tokens']/(r['e2e_ms']/1e3)))
    a = r['agents']['1:0']; print('1:0 out', a['output'][:12], [round(x,2) for x in a['logprobs'][:6]])
    eng.close()
