"""Per-agent teacher-forced logit error of one request (debug):
python tools/logit_err.py CONFIG SAMPLE [MODE]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.configs import models_of  # noqa: E402
from oracle.parity import check_agent  # noqa: E402
from paper_2512_18126_b200 import capi  # noqa: E402
from paper_2512_18126_b200.configs import CONFIGS, agent_tag  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1]])
if len(sys.argv) > 3:
    cfg["mode"] = sys.argv[3]
eng, qc = capi.engine_for(cfg, keep_logits=True)
g = eng.run_query(qc, sample=int(sys.argv[2]))
models = models_of(cfg, 1024)
for name, ga in sorted(g["agents"].items()):
    if not ga["output"]:
        continue
    a = tuple(int(x) for x in name.split(":"))
    L = np.stack([eng.read_logits(a, k) for k in range(len(ga["output"]))])
    chk = check_agent(models[agent_tag(cfg, *a)], ga["prompt"], ga["output"], ga["logprobs"], gpu_logits=L)
    print(name, len(ga["prompt"]), {k: chk[k] for k in ("checked", "skipped_near_tie", "max_lp_err", "max_logit_err", "lp_ok")})
eng.close()
