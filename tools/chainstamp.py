"""Decode-chain timeline from in-kernel %globaltimer stamps (chain.py):
python tools/chainstamp.py [config] [first_tick_frac] [out_tokens] [json]"""
import json
import sys

sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi, chain
from paper_2512_18126_b200.configs import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else 'C1'
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.75
cfg = dict(CONFIGS[name])
if len(sys.argv) > 3:
    cfg['out_len'] = [int(sys.argv[3])] * 3
eng, qc = capi.engine_for(cfg)
for i in range(2):
    eng.run_query(qc, sample=0, resolve=False, detail=False)
recs, e2e = chain.collect(eng, qc, 0)
tl = chain.timeline(chain.ticks(recs), frac)
print(name, 'records', len(recs), 'stamped e2e_ms %.2f' % e2e)
print('median tick %.2f us, gap to next tick %.2f us, %d ticks' % (tl['tick_us'], tl['gap_to_next_tick_us'], tl['ticks_analysed']))
print('%-16s %8s %8s %8s %8s' % ('kernel', 'start', 'release', 'end', 'rel->end'))
for k in tl['kernels']:
    print('%-16s %8.2f %8.2f %8.2f %8.2f' % (k['kernel'], k['start_us'], k['release_us'], k['end_us'], k['release_to_end_us']))
if len(sys.argv) > 4:
    print(json.dumps(tl))
