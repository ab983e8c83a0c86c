"""tcgen05 prefill GEMM vs torch.matmul (debug timing):
python tools/gemm_time.py M N K [reps]   (out fp32 = A . W^T, bf16 operands)"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18126_b200 import capi  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
W = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
out = torch.empty(M, N, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


ours = timed(lambda: capi.check(capi.lib().moa_k_gemm_tc(A.data_ptr(), M, W.data_ptr(), N, K, out.data_ptr(), 0)))
ref = timed(lambda: torch.matmul(A, W.T))
fl = 2.0 * M * N * K
err = float((out - (A.float() @ W.float().T)).abs().max())
print(f"M{M} N{N} K{K}: ours {ours * 1e3:.1f} us {fl / ours / 1e9:.0f} TFLOP/s | torch {ref * 1e3:.1f} us "
      f"{fl / ref / 1e9:.0f} TFLOP/s | ratio {ref / ours:.2f} | max err {err:.2e}")
