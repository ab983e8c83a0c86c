"""gemv_tc launched alone (synchronised between launches) at the 1b shapes,
with per-CTA %globaltimer stamps: start, TMEM ready, first tile landed,
MMAs done, end."""
import sys
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
L = capi.lib()
tr = torch.zeros(4096 * 8, dtype=torch.int64, device='cuda')
L.moa_k_debug_trace(tr.data_ptr())
for (N, K) in ((3072, 2048), (2048, 2048), (16384, 2048), (2048, 8192)):
    W = (torch.randn(N, K, device='cuda') * 0.02).to(torch.bfloat16)
    A = torch.randn(16, K, device='cuda').to(torch.bfloat16)
    out = torch.empty(8, N, device='cuda')
    st = torch.cuda.current_stream().cuda_stream
    for i in range(4):
        tr.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        capi.check(L.moa_k_gemv_tc(A.data_ptr(), 8, W.data_ptr(), N, K, out.data_ptr(), st))
        e1.record()
        torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(-1, 8)
    t = t[t[:, 0] > 0]
    # SM cycle counters (not comparable across SMs): intervals relative to each CTA's own start, in us @1.965 GHz
    rel = np.where(t[:, :7] > 0, (t[:, :7] - t[:, :1]) / 1965.0, np.nan)
    sm = t[:, 7]
    per_sm = np.bincount(sm.astype(np.int64))
    print(f'N={N} K={K} ctas={len(t)} event_ms={e0.elapsed_time(e1):.4f} | start max {rel[:,0].max():.1f} | tmem max {rel[:,1].max():.1f} '
          f'| first tile med {np.median(rel[:,2]):.1f} max {rel[:,2].max():.1f} | mma done med {np.median(rel[:,3]):.1f} max {rel[:,3].max():.1f} '
          f'| end med {np.median(rel[:,4]):.1f} max {rel[:,4].max():.1f} | sms used {np.count_nonzero(per_sm)} max ctas/sm {per_sm.max()}')
    last = ~np.isnan(rel[:, 6])
    print('   nonzero per slot', [(t[:, k] > 0).sum() for k in range(8)])
    if not last.any():
        continue
    med = [np.nanmedian(rel[last][:, k]) for k in (3, 5, 6, 4)]
    print('   last arrivers: n %d mma done med %.1f atomic-ret med %.1f loads-done med %.1f end med %.1f max %.1f' % (last.sum(), *med, np.nanmax(rel[last][:, 4])))
    slow = np.argsort(-np.nan_to_num(rel[:, 4]))[:3]
    for i in slow:
        print('   slow cta', i, 'sm', sm[i], 'stamps', np.round(rel[i], 1))
L.moa_k_debug_trace(0)
