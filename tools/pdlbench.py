"""Chains of gemv_tc launches (1b shapes) in a CUDA graph: per-kernel time,
to see whether programmatic dependent launch overlaps consecutive kernels."""
import os, sys
import torch
sys.path.insert(0, '/root/repo')
from paper_2512_18126_b200 import capi
L = capi.lib()
n_chain = 40
for (N, K) in ((3072, 2048), (2048, 8192), (16384, 2048)):
    Ws = [(torch.randn(N, K, device='cuda') * 0.02).to(torch.bfloat16) for _ in range(4)]
    A = torch.randn(16, K, device='cuda').to(torch.bfloat16)
    out = torch.empty(8, N, device='cuda')
    s = torch.cuda.Stream()
    def chain():
        st = torch.cuda.current_stream().cuda_stream
        for i in range(n_chain):
            capi.check(L.moa_k_gemv_tc(A.data_ptr(), 8, Ws[i % 4].data_ptr(), N, K, out.data_ptr(), st))
    with torch.cuda.stream(s):
        chain()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        chain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (10 * n_chain)
    mb = N * K * 2 / 1e6
    print(f"N={N} K={K} PDL={'off' if os.environ.get('MOA_NO_PDL') == '1' else 'on'} graph chain: {us:.2f} us/kernel, {mb / us * 1e-3 * 1e3:.0f} GB/s")

# the floor: a graph of trivial PDL kernels
cnt = torch.zeros(1, dtype=torch.int32, device='cuda')
for ctas in (1, 148):
    s = torch.cuda.Stream()
    def chain():
        st = torch.cuda.current_stream().cuda_stream
        for i in range(n_chain):
            capi.check(L.moa_k_noop(cnt.data_ptr(), ctas, st))
    with torch.cuda.stream(s):
        chain()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        chain()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"noop chain, {ctas} CTAs, PDL={'off' if os.environ.get('MOA_NO_PDL') == '1' else 'on'}: {e0.elapsed_time(e1) * 1e3 / (10 * n_chain):.2f} us/kernel")
