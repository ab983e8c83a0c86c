"""Incremental-prefill chunk-tick microbenchmark: one agent of <shape> holds a
P-token prompt, then every tick appends one <rows>-token chunk
(`prefill_only`, the successor side of the pipelined overlap).  Prints the
device time per chunk tick (tick events) and, from a second pass with probes
(events around every launch, graphs bypassed), the per-kind split:

    python tools/chunkbench.py 8b 32 2048 [chunks]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.rng import synth_tokens  # noqa: E402
from paper_2512_18126_b200 import capi  # noqa: E402

shape, rows, P = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
N = min(int(sys.argv[4]) if len(sys.argv) > 4 else 24, (8000 - P) // rows)
eng = capi.Engine([capi.model_spec("m", shape, 1, max_agents=2)], max_ctx=P + rows * N + 64, max_out=8)


def run(probe=False):
    eng.reset()
    eng.add_agent((2, 0), 0)
    eng.prefill_only((2, 0), 0, synth_tokens(0, "p", P))
    eng.step()
    eng.trace(True)
    eng.probe(probe)
    eng.mark_start()
    t0 = eng.tick()
    for c in range(N):
        eng.prefill_only((2, 0), P + c * rows, synth_tokens(c, "c", rows))
        eng.step()
    t1 = eng.tick()
    return t0, t1


run()
t0, t1 = run()
ts = np.array([eng.tick_seconds(t) for t in range(t0, t1)]) * 1e3
d = np.diff(ts)
spec = eng.models[0]
wb = 2.0 * ((spec.n_heads + 2 * spec.n_kv_heads) * spec.head_dim * spec.d + spec.d * spec.n_heads * spec.head_dim
            + 3 * spec.ffn * spec.d) * spec.n_layers
print(f"{shape} chunk rows={rows} ctx={P}: chunk tick p50 {np.median(d):.3f} ms p10 {np.percentile(d, 10):.3f} "
      f"p90 {np.percentile(d, 90):.3f}; layer weights {wb / 1e9:.2f} GB -> {wb / np.median(d) / 1e6:.0f} GB/s")
run(probe=True)
st = eng.probe_stats()
eng.probe(False)
tot = sum(v["ms"] for v in st.values())
for k, v in st.items():
    if v["launches"]:
        print(f"  {k:12s} launches {v['launches']:5d} ms/chunk {v['ms'] / N:7.3f} avg us {1e3 * v['ms'] / v['launches']:8.2f} "
              f"GB/s {v['bytes'] / (v['ms'] * 1e6):7.0f}")
print(f"  probed total ms/chunk {tot / N:.3f}")
eng.close()
