"""Per-tick device time of a request (engine tracing): where the e2e goes.
python tools/ticktime.py C1 [out_len]"""
import os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS

name = sys.argv[1]
cfg = dict(CONFIGS[name])
if len(sys.argv) > 2 and int(sys.argv[2]):
    cfg['out_len'] = [int(sys.argv[2])] * 3
eng, qc = capi.engine_for(cfg)
eng.trace(True)
for i in range(3):
    r = eng.run_query(qc, sample=0, resolve=False, detail=True, trace=True)
t = np.array(r['tick_ms'])
d = np.diff(np.concatenate([[0.0], t]))
print(name, 'e2e_ms %.2f host_ms %.2f ticks %d' % (r['e2e_ms'], r['host_ms'], r['ticks']))
print('tick ms: p10 %.4f p50 %.4f p90 %.4f max %.4f sum %.2f' % tuple(list(np.percentile(d, [10, 50, 90])) + [d.max(), d.sum()]))
order = np.argsort(-d)[:12]
print('slowest ticks:', ' '.join('%d:%.3f' % (k, d[k]) for k in order))
ag = r['agents']
for k, a in sorted(ag.items()):
    print(k, 'decode [%d,%d) complete %d prompt %d out %d pruned %d' % (a['decode_start'], a['decode_end'], a['complete'], a['prompt_tokens'], a['output_tokens'], a['pruned']))
print('deltas', ' '.join('%.3f' % x for x in d))
