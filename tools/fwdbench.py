"""Decode-forward microbenchmark: one model, R agents at a ~C-token context,
device time per decode tick (engine tick events) and the weight-stream rate.

    python tools/fwdbench.py 8b 4 2048 [ticks]
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18126_b200 import capi  # noqa: E402
from oracle.rng import synth_tokens  # noqa: E402

shape, R, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
T = int(sys.argv[4]) if len(sys.argv) > 4 else 64
eng = capi.Engine([capi.model_spec("m", shape, 1, max_agents=R)], max_ctx=ctx + T + 64, max_out=T + 8)
for r in range(R):
    eng.add_agent((1, r), 0)
    eng.generate((1, r), synth_tokens(r, "p", ctx), T, 32)
eng.trace(True)
eng.mark_start()
t0 = eng.tick()
busy = True
while busy:
    _, busy = eng.step()
t1 = eng.tick()
ts = np.array([eng.tick_seconds(t) for t in range(t0, t1)]) * 1e3
d = np.diff(ts)
spec = eng.models[0]
wb = 2.0 * ((spec.n_heads + 2 * spec.n_kv_heads) * spec.head_dim * spec.d + spec.d * spec.n_heads * spec.head_dim
            + 3 * spec.ffn * spec.d) * spec.n_layers + 2.0 * spec.vocab * spec.d
dec = d[2:]
med = float(np.median(dec))
kv = 4.0 * spec.n_layers * spec.n_kv_heads * spec.head_dim * R * (ctx + T / 2)
print(f"{shape} R={R} ctx={ctx}: first tick {ts[0]:.2f} ms, decode tick p50 {med:.4f} ms p10 {np.percentile(dec, 10):.4f} "
      f"p90 {np.percentile(dec, 90):.4f}; weights {wb / 1e9:.3f} GB + kv {kv / 1e9:.3f} GB -> "
      f"{(wb + kv) / med / 1e6:.0f} GB/s")
eng.close()
