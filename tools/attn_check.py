"""Attention kernel hook vs fp32 torch on the parity test's tick (debug):
python tools/attn_check.py nh nkv hd max_ctx mode [reps]"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18126_b200 import capi  # noqa: E402

nh, nkv, hd, max_ctx, mode = (int(x) for x in sys.argv[1:6])
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 1
g = torch.Generator(device="cpu").manual_seed(7 + nh + hd)
slots = 4
kv_stride = nkv * max_ctx * hd
kpool = (torch.randn(slots * kv_stride, generator=g) * 0.5).to(torch.bfloat16).cuda()
vpool = torch.randn(slots * kv_stride, generator=g).to(torch.bfloat16).cuda()
late = max_ctx - 200
rows = [(0, p) for p in range(100, 230)] + [(1, p) for p in range(0, 70)] + [(2, late)] + \
       [(3, p) for p in range(10, 20)] + [(3, p) for p in range(40, 45)] + [(1, late + 150)]
R = len(rows)
q = torch.randn(R, nh, hd, generator=g).to(torch.bfloat16).cuda()
rd = torch.tensor([[kv, pos, 0, 0] for kv, pos in rows], dtype=torch.int32).cuda()
meta = torch.tensor([R, 0, max(p for _, p in rows)], dtype=torch.int32).cuda()
K = kpool.float().view(slots, nkv, max_ctx, hd)
V = vpool.float().view(slots, nkv, max_ctx, hd)
ref = torch.empty(R, nh, hd, device="cuda")
for i, (kv, pos) in enumerate(rows):
    for h in range(nh):
        kh = h // (nh // nkv)
        sc = (q[i, h].float() @ K[kv, kh, :pos + 1].T) / math.sqrt(hd)
        ref[i, h] = torch.softmax(sc, -1) @ V[kv, kh, :pos + 1]
worst = 0.0
for _ in range(reps):
    out = torch.zeros(R, nh, hd, dtype=torch.bfloat16, device="cuda")
    capi.check(capi.lib().moa_k_attention(q.data_ptr(), rd.data_ptr(), R, meta.data_ptr(), nh, nkv, hd,
                                          kpool.data_ptr(), vpool.data_ptr(), kv_stride, max_ctx, out.data_ptr(),
                                          mode, 0, slots))
    torch.cuda.synchronize()
    d = (out.float() - ref).abs()
    err = float(d.max())
    if err > worst:
        worst = err
        bad = (d.amax(dim=(1, 2)) > 2e-2).nonzero().flatten().tolist()
        print(f"err {err:.4f} bad rows {[(i, rows[i]) for i in bad[:8]]} n_bad {len(bad)}")
print(f"mode {mode}: worst {worst:.4f} over {reps} reps")
