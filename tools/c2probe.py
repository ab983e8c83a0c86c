"""C2 (1b agents) per-kernel breakdown: device time per request and the
per-kernel probes (CUDA events around each launch, graphs bypassed)."""
import json, sys
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import C2
out = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = dict(C2, out_len=[out, out, out])
eng, qc = capi.engine_for(cfg)
for i in range(2):
    r = eng.run_query(qc, sample=i, resolve=False, detail=False)
    print('graphs: e2e_ms', round(r['e2e_ms'], 2), 'ticks', r['ticks'], 'fwd', r['forwards'], 'rows', r['rows'],
          'host_ms', round(r['host_ms'], 2), 'ms/tick', round(r['e2e_ms'] / r['ticks'], 3), flush=True)
eng.probe(True)
r = eng.run_query(qc, sample=0, resolve=False, detail=False)
st = eng.probe_stats()
eng.probe(False)
tot = sum(v['ms'] for v in st.values())
print('probed e2e_ms', round(r['e2e_ms'], 2), 'sum kernel ms', round(tot, 2))
for k, v in st.items():
    print(f"{k:10s} n={v['launches']:6d} ms={v['ms']:9.2f} avg_us={1e3*v['ms']/max(1,v['launches']):8.2f} "
          f"GB/s={v['bytes']/max(1e-12,v['ms']/1e3)/1e9:8.1f}")
