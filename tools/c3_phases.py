"""Where a tree request's device time goes: per tree layer, the span from the
first prefill to the last completion, its ticks and their mean duration
(engine tick events, device clock):

    python tools/c3_phases.py [C3] [sample]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18126_b200 import capi  # noqa: E402
from paper_2512_18126_b200.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
sample = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS[name]
eng, qc = capi.engine_for(cfg)
eng.trace(True)
eng.run_query(qc, sample=sample, resolve=False, detail=False)  # warm: graphs captured
r = eng.run_query(qc, sample=sample, resolve=False, detail=False, trace=True)
tick_end = np.array(r["tick_ms"])  # device ms at the end of each tick
tv = r["trace_view"]
print(f"{name} sample {sample}: e2e {r['e2e_ms']:.1f} ms, {len(tick_end)} ticks, tokens {r['tokens']}")
prev_end = 0.0
for layer in sorted({a["layer"] for a in tv["agents"]}):
    ags = [a for a in tv["agents"] if a["layer"] == layer and a["invoked"]]
    if not ags:
        continue
    start = min(min((p[0] for p in a["prefill"]), default=a["complete_t"]) for a in ags) * 1e3
    end = max(a["complete_t"] for a in ags) * 1e3
    ticks = tick_end[(tick_end > prev_end) & (tick_end <= end)]
    d = np.diff(np.concatenate([[prev_end], ticks]))
    tags = sorted({a["model_tag"] for a in ags})
    print(f"layer {layer}: {len(ags)} agents {tags}: first prefill {start:8.1f} ms, last completion {end:8.1f} ms; "
          f"{len(ticks)} ticks after the previous layer, mean {d.mean() if len(d) else 0:.3f} ms, "
          f"p50 {np.median(d) if len(d) else 0:.3f}, max {d.max() if len(d) else 0:.2f}, sum {d.sum():.1f}")
    big = np.argsort(d)[-5:][::-1]
    print("   longest ticks:", ", ".join(f"{d[i]:.2f} ms @ {ticks[i]:.0f}" for i in big))
    prev_end = end
eng.close()
