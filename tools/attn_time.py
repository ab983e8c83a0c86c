"""Prefill attention kernels on a prompt-prefill tick (debug timing):
python tools/attn_time.py nh nkv hd agents prompt [mode ...]
Rows: `agents` prompts of `prompt` tokens each (one run per agent); modes as
moa_k_attention (17: mma.sync prefill, 25: tcgen05 prefill; no per-row kernel:
every row is in a run).  Device time per call
(CUDA events, median of 10) and the causal flops rate."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18126_b200 import capi  # noqa: E402

nh, nkv, hd, A, Pn = (int(x) for x in sys.argv[1:6])
modes = [int(x) for x in sys.argv[6:]] or [17, 25]
max_ctx = ((Pn + 255) // 256) * 256
kv_stride = nkv * max_ctx * hd
g = torch.Generator(device="cpu").manual_seed(1)
kpool = (torch.randn(A * kv_stride, generator=g) * 0.5).to(torch.bfloat16).cuda()
vpool = torch.randn(A * kv_stride, generator=g).to(torch.bfloat16).cuda()
rows = [(a, p) for a in range(A) for p in range(Pn)]
R = len(rows)
q = torch.randn(R, nh, hd, generator=g).to(torch.bfloat16).cuda()
rd = torch.tensor([[kv, pos, 0, 0] for kv, pos in rows], dtype=torch.int32).cuda()
meta = torch.tensor([R, 0, Pn - 1], dtype=torch.int32).cuda()
flops = 4.0 * hd * nh * A * Pn * (Pn + 1) / 2
outs = {}
for mode in modes:
    out = torch.zeros(R, nh, hd, dtype=torch.bfloat16, device="cuda")
    ts = []
    for it in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        capi.check(capi.lib().moa_k_attention(q.data_ptr(), rd.data_ptr(), R, meta.data_ptr(), nh, nkv, hd,
                                              kpool.data_ptr(), vpool.data_ptr(), kv_stride, max_ctx, out.data_ptr(),
                                              mode, 0, A))
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    outs[mode] = out.float()
    print(f"mode {mode}: {ms * 1e3:.1f} us  {flops / ms / 1e9:.1f} TFLOP/s")
if len(outs) > 1:
    ms_ = list(outs.values())
    print("max |diff| between modes:", float((ms_[0] - ms_[1]).abs().max()))
