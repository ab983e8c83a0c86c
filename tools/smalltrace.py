"""Step timeline (layer 1; CTA clock us from kernel start) of the
cluster-resident small-agent forward inside a C1 request."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
L = capi.lib()
cfg = dict(CONFIGS['C1'], out_len=[16, 16, 16])
eng, qc = capi.engine_for(cfg)
eng.run_query(qc, sample=0, resolve=False, detail=False)
tr = torch.zeros(16 * 64, dtype=torch.int64, device='cuda')
L.moa_k_debug_trace_small(tr.data_ptr())
eng.run_query(qc, sample=1, resolve=False, detail=False)
torch.cuda.synchronize()
L.moa_k_debug_trace_small(0)
t = tr.cpu().numpy().reshape(16, 64)
rel = (t - t[:, :1]) / 1965.0
names = {0: 'start', 1: 'pdl_wait', 2: 'embed+csync', 20: 'attn done', 21: 'attn csync', 22: 'layers done'}
for j, nm in enumerate(['qkv', 'o', 'gu', 'down']):
    names[3 + 4 * j] = nm + ' slab ready'
    names[4 + 4 * j] = nm + ' gemv done'
    names[5 + 4 * j] = nm + ' bcast done'
    names[6 + 4 * j] = nm + ' csync'
for ev in sorted(names, key=lambda e: np.median(rel[:, e])):
    col = rel[:, ev]
    print(f'{names[ev]:18s} med {np.median(col):7.2f} max {col.max():7.2f}')
