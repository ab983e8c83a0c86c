"""Per-CTA timeline (SM clock, us @1.965GHz from each CTA's start) of the
persistent LM head inside a real C1 request."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
from paper_2512_18126_b200.configs import CONFIGS
L = capi.lib()
name = sys.argv[1] if len(sys.argv) > 1 else 'C1'
cfg = dict(CONFIGS[name], out_len=[8, 8, 8])
eng, qc = capi.engine_for(cfg)
tr = torch.zeros(4096 * 8, dtype=torch.int64, device='cuda')
eng.run_query(qc, sample=0, resolve=False, detail=False)
L.moa_k_debug_trace(tr.data_ptr())
eng.run_query(qc, sample=1, resolve=False, detail=False)
torch.cuda.synchronize()
L.moa_k_debug_trace(0)
t = tr.cpu().numpy().reshape(-1, 8)[:148]
rel = np.where(t[:, :6] > 0, (t[:, :6] - t[:, :1]) / 1965.0, np.nan)
for k, nm in enumerate(['start', 'first tile', 'mma done', 'epi done', 'atomic', 'merge end']):
    col = rel[:, k]
    print(f'{nm:10s} med {np.nanmedian(col):6.2f} max {np.nanmax(col):6.2f} n {np.count_nonzero(~np.isnan(col))}')
