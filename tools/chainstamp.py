"""Decode-chain timeline from in-kernel %globaltimer stamps (stamp.cuh):
per kernel of a tick, when its CTAs start, when the PDL wait releases, the
intermediate phases and the end -- averaged over the ticks of one phase of a
C1 request.  python tools/chainstamp.py [config] [first_tick_frac]"""
import collections
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS

NAMES = {0x40000: 'o_gate_up', 0x10010: 'o_proj', 0x12010: 'gate_up', 0x11040: 'down', 0x10040: 'down', 0x20000: 'qkv_attn', 0x20001: 'qkv_attn0',
         0x30000: 'lm_head'}
name = sys.argv[1] if len(sys.argv) > 1 else 'C1'
eng, qc = capi.engine_for(dict(CONFIGS[name]))
for i in range(2):
    eng.run_query(qc, sample=0, resolve=False, detail=False)
cap = 1 << 22
buf = torch.zeros(2 + 2 * cap, dtype=torch.int64, device='cuda')
capi.lib().moa_k_chain_stamp(buf.data_ptr())
r = eng.run_query(qc, sample=0, resolve=False, detail=False)
torch.cuda.synchronize()
capi.lib().moa_k_chain_stamp(0)
n = int(buf[0].item())
rec = buf[2:2 + 2 * min(n, cap)].view(-1, 2).cpu().numpy().astype(np.uint64)
meta, t = rec[:, 0], rec[:, 1].astype(np.int64)
tag = (meta >> np.uint64(32)).astype(np.int64)
phase = ((meta >> np.uint64(24)) & np.uint64(0xff)).astype(np.int64)
t = t - t.min()
print(name, 'records', n, 'e2e_ms %.2f ticks %d' % (r['e2e_ms'], r['ticks']))
# instances: per tag, phase-0 stamps clustered by gaps > 3 us
inst = []
for tg in np.unique(tag):
    e = np.sort(t[(tag == tg) & (phase == 0)])
    if len(e) == 0:
        continue
    cuts = np.where(np.diff(e) > 3000)[0]
    starts = np.split(e, cuts + 1)
    for s in starts:
        inst.append(dict(tag=int(tg), t0=int(s.min()), ph=collections.defaultdict(list)))
inst.sort(key=lambda d: d['t0'])
by_tag = collections.defaultdict(list)
for k, d in enumerate(inst):
    by_tag[d['tag']].append(k)
for tg, ks in by_tag.items():
    t0s = np.array([inst[k]['t0'] for k in ks])
    m = tag == tg
    for tt, ph in zip(t[m], phase[m]):
        j = np.searchsorted(t0s, tt, side='right') - 1
        if j >= 0:
            inst[ks[j]]['ph'][int(ph)].append(int(tt))
# ticks end at lm_head instances
ticks, cur = [], []
for d in inst:
    cur.append(d)
    if d['tag'] == 0x30000:
        ticks.append(cur)
        cur = []
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.75
sel = ticks[int(len(ticks) * frac):-1]
print('ticks seen', len(ticks), 'analysed', len(sel), 'kernels/tick', collections.Counter(len(x) for x in sel))
L = collections.Counter(len(x) for x in sel).most_common(1)[0][0]
sel = [x for x in sel if len(x) == L]
rows = []
for pos in range(L):
    vals = collections.defaultdict(list)
    for k, tk in enumerate(sel):
        d = tk[pos]
        base = tk[0]['t0']
        prev_end = max(tk[pos - 1]['ph'][2]) if pos > 0 and tk[pos - 1]['ph'][2] else None
        vals['start'].append(d['t0'] - base)
        for ph, ts in d['ph'].items():
            vals['p%d_max' % ph].append(max(ts) - base)
            vals['p%d_min' % ph].append(min(ts) - base)
        if prev_end is not None and d['ph'][1]:
            vals['release_after_prev_end'].append(max(d['ph'][1]) - prev_end)
    rows.append((NAMES.get(tk[pos]['tag'], hex(tk[pos]['tag'])), {k: float(np.median(v)) for k, v in vals.items()}))
tick_len = np.median([max(tk[-1]['ph'][2]) - tk[0]['t0'] for tk in sel])
gap = np.median([sel[i + 1][0]['t0'] - max(sel[i][-1]['ph'][2]) for i in range(len(sel) - 1)])
print('median tick: first entry -> lm_head end %.2f us; lm end -> next tick first entry %.2f us' % (tick_len / 1e3, gap / 1e3))
print('%-10s %8s %8s %8s %8s %8s %8s %8s %8s %8s %8s' % ('kernel', 'start', 'wait_rel', 'p3', 'p4', 'p5', 'p6', 'p7', 'end_max', 'dur', 'rel-prev'))
for nm, v in rows:
    def g(k):
        return '%8.2f' % (v[k] / 1e3) if k in v else '%8s' % '-'
    dur = (v.get('p2_max', 0) - v.get('p1_max', 0)) / 1e3
    print('%-10s %s %s %s %s %s %s %s %s %8.2f %s' % (nm, g('start'), g('p1_max'), g('p3_max'), g('p4_max'), g('p5_max'),
                                                   g('p6_max'), g('p7_max'), g('p2_max'), dur, g('release_after_prev_end')))
    if nm == 'lm_head':
        print('  lm_head min-over-CTAs: wait %s staged %s mma_start %s mma_issued %s tiles %s end %s' % (
            g('p1_min'), g('p3_min'), g('p5_min'), g('p7_min'), g('p4_min'), g('p2_min')))
