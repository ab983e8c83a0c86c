"""In-graph decode-tick timeline (chain.py stamps) of R same-model agents at a
~P-token context, driven through the engine protocol:
python tools/chaindec.py <shape> <R> <P> [ticks]"""
import collections
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.rng import synth_tokens  # noqa: E402
from paper_2512_18126_b200 import capi, chain  # noqa: E402

shape, R, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
T = int(sys.argv[4]) if len(sys.argv) > 4 else 48
eng = capi.Engine([capi.model_spec("m", shape, 1, max_agents=R)], max_ctx=P + T + 64, max_out=T + 8)


def run():
    eng.reset()
    for r in range(R):
        eng.add_agent((1, r), 0)
        eng.generate((1, r), synth_tokens(r, "p", P), T, 32)
    busy = True
    while busy:
        _, busy = eng.step()


run()  # warm: graphs captured
import torch  # noqa: E402
cap = 1 << 24
buf = torch.zeros(2 + 2 * cap, dtype=torch.int64, device="cuda")
capi.check(capi.lib().moa_k_chain_stamp(buf.data_ptr()))
run()
torch.cuda.synchronize()
capi.lib().moa_k_chain_stamp(0)
n = min(int(buf[0].item()), cap)
rec = buf[2:2 + 2 * n].view(-1, 2).cpu().numpy().astype(np.uint64)
meta, t = rec[:, 0], rec[:, 1].astype(np.int64)
recs = np.stack([(meta >> np.uint64(32)).astype(np.int64), ((meta >> np.uint64(24)) & np.uint64(0xff)).astype(np.int64),
                 (meta & np.uint64(0xffffff)).astype(np.int64), t - t.min()], axis=1)
cnt = collections.Counter((chain._name(int(a)), int(b)) for a, b in zip(recs[:, 0], recs[:, 1]))
print(shape, R, P, "records", n, dict(sorted(cnt.items())))
L = {"tiny": 4, "1b": 16, "8b": 32}[shape]
recs = recs[np.argsort(recs[:, 3], kind="stable")]  # time order: each tick is one contiguous slice
tag_all, ph_all, tt_all = recs[:, 0], recs[:, 1], recs[:, 3]
tag, ph, tt = tag_all, ph_all, tt_all
LM = 0x30000
lm_end = np.sort(tt_all[(tag_all == LM) & (ph_all == 2)])
# LM head instances: cluster CTA end stamps (one instance per tick)
ends = [s_.max() for s_ in np.split(lm_end, np.where(np.diff(lm_end) > 5000)[0] + 1)]
per_tag_launch = {}
rows = collections.defaultdict(list)  # (layer position, name) -> incremental us
phases = collections.defaultdict(lambda: collections.defaultdict(list))
ticks = 0
for k in range(len(ends) // 3, len(ends) - 1):  # steady-state decode ticks
    lo, hi = ends[k], ends[k + 1]
    i0, i1 = np.searchsorted(tt_all, lo, side="right"), np.searchsorted(tt_all, hi, side="right")
    tag, ph, tt = tag_all[i0:i1], ph_all[i0:i1], tt_all[i0:i1]
    m = np.ones(len(tt), bool)
    insts = []
    for tg in np.unique(tag[m]):
        e = np.sort(tt[m & (tag == tg) & (ph == 0)])
        if len(e) == 0:
            continue
        n_inst = 1 if tg == LM else (2 * L if chain._name(int(tg)) == "rmsnorm" else L)
        if len(e) < n_inst:
            continue
        gaps = np.diff(e)
        cut = np.sort(np.argsort(gaps)[::-1][: n_inst - 1]) + 1
        for grp in np.split(e, cut):
            a, b = grp.min(), grp.max()
            sel = m & (tag == tg) & (tt >= a)
            insts.append((int(a), int(tg)))
    insts.sort()
    # end of each instance: max phase-2 stamp of its CTAs between its start and the next same-tag start
    by_tag = collections.defaultdict(list)
    for a, tg in insts:
        by_tag[tg].append(a)
    inst_end = {}
    for tg, starts in by_tag.items():
        starts = sorted(starts) + [hi + 1]
        e2 = np.sort(tt[m & (tag == tg) & (ph == 2)])
        for j in range(len(starts) - 1):
            w = e2[(e2 >= starts[j]) & (e2 < starts[j + 1])]
            inst_end[(tg, starts[j])] = int(w.max()) if len(w) else starts[j]
    prev = lo
    per_layer = len(insts) // L if L else 1
    for j, (a, tg) in enumerate(insts):
        e_ = inst_end[(tg, a)]
        key = (j % per_layer if tg != LM else 99, chain._name(int(tg)))
        rows[key].append((e_ - prev) / 1e3)
        # phase profile of this launch relative to the previous launch's end:
        # per phase, the median and the max over its CTAs
        mm = m & (tag == tg) & (tt >= a) & (tt <= e_)
        for p_ in range(8):
            v = tt[mm & (ph == p_)]
            if len(v):
                phases[key][p_].append(((np.median(v) - prev) / 1e3, (v.max() - prev) / 1e3))
        prev = max(prev, e_)
    ticks += 1
tag, ph, tt = tag_all, ph_all, tt_all
print(f"{ticks} steady ticks; tick median {np.median(np.diff(ends[len(ends)//3:])) / 1e3:.1f} us")
tot = 0.0
for key in sorted(rows):
    v = rows[key]
    per_tick = float(np.sum(v)) / ticks
    tot += per_tick
    print(f"  pos {key[0]:3d} {key[1]:28s} n/tick={len(v)/ticks:5.1f} median incr {np.median(v):7.2f} us  per tick {per_tick:8.1f} us")
print(f"  sum {tot:.1f} us")
print("phase stamps (us after the previous launch's end): median CTA / last CTA")
for key in sorted(phases):
    cells = []
    for p_, v in sorted(phases[key].items()):
        a_ = np.median([x[0] for x in v])
        b_ = np.median([x[1] for x in v])
        cells.append(f"p{p_}:{a_:6.2f}/{b_:6.2f}")
    print(f"  pos {key[0]:3d} {key[1]:26s} " + "  ".join(cells))
eng.close()
