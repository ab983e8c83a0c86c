"""Raw launch sequence from chain stamps (chain.py) over a window of a
request: python tools/chaindump.py CONFIG OUT_TOKENS FIRST COUNT"""
import sys

sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi, chain
from paper_2512_18126_b200.configs import CONFIGS

cfg = dict(CONFIGS[sys.argv[1]])
cfg['out_len'] = [int(sys.argv[2])] * 3
eng, qc = capi.engine_for(cfg)
eng.run_query(qc, sample=0, resolve=False, detail=False)
recs, e2e = chain.collect(eng, qc, 0)
ticks = chain.ticks(recs)
inst = [d for tk in ticks for d in tk]
a, n = int(sys.argv[3]), int(sys.argv[4])
prev_end = None
print('e2e %.2f ms, %d launches' % (e2e, len(inst)))
print('%-28s %10s %9s %9s %9s %9s' % ('kernel', 'start', 'release', 'end', 'rel-prev', 'rel->end'))
for d in inst[a:a + n]:
    rel = max(d['ph'][1]) / 1e3 if d['ph'][1] else float('nan')
    end = chain._end(d) / 1e3
    print('%-28s %10.2f %9.2f %9.2f %9.2f %9.2f' % (chain._name(d['tag']), d['t0'] / 1e3, rel, end,
                                                    rel - prev_end if prev_end else float('nan'), end - rel))
    prev_end = end
