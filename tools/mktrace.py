"""Phase timeline of one persistent decode forward (decode_mk.cu stamps).
Per phase: when the grid barrier released the X writers (min/max over CTAs),
staging done, first MMA, first epilogue, last CTA's arrival."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else 'C2'
out = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg = dict(CONFIGS[name], out_len=[out] * 3)
eng, qc = capi.engine_for(cfg)
for m in range(len(cfg['models'])):
    eng.megakernel(m, True, True)
r = eng.run_query(qc, sample=0, resolve=False, detail=False)
print(name, 'e2e_ms', r['e2e_ms'], 'ticks', r['ticks'])
tr = eng.mk_trace(0).astype(np.int64)
G = 148
P = tr.size // (G * 8)
t = tr.reshape(P, G, 8)
t0 = t[0, :, 5][t[0, :, 5] > 0].min()
kinds = ['EMB'] + [k for _ in range((P - 3) // 5) for k in ('QKV', 'ATT', 'O', 'GU', 'DN')] + ['LM', 'LMX']
prev_done = t0
tot = {}
for p in range(P):
    def col(e):
        v = t[p, :, e]
        v = v[v > 0]
        return ((v.min() - t0), (v.max() - t0)) if v.size else (None, None)
    w0 = col(0); x1 = col(1); m2 = col(2); e3 = col(3); a4 = col(4); t6 = col(6); m7 = col(7)
    done = a4[1]
    dur = done - (prev_done - t0)
    tot[kinds[p]] = tot.get(kinds[p], 0) + dur
    if p < 12 or p >= P - 3:
        f = lambda x: '(%s)' % ','.join('-' if v is None else '%.1f' % (v / 1e3) for v in x)
        print(f"{p:3d} {kinds[p]:4s} release {f(w0)} staged {f(x1)} mma {f(m2)} mma_end {f(m7)} epi1 {f(e3)} arrive {f(a4)}  phase_us {dur/1e3:.2f}")
    prev_done = done + t0
print('total us', (prev_done - t0) / 1e3, {k: round(v / 1e3, 1) for k, v in tot.items()})
