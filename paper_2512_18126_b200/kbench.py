"""Kernel roofline microbenchmarks at the `1b` / `8b` agent shapes.

    python -m paper_2512_18126_b200.kbench [--json out.json]

* decode GEMV (HBM-bound): y = x . W^T for the 1b layer matrices and LM head
  with R = 1..8 rows; weights cycle through 16 layer copies (> 126 MB L2),
  so every launch streams from HBM.  achieved = algorithmic bytes / time.
* prefill GEMM on tcgen05 (tensor-bound): M = 512 / 2048 rows x the 1b
  gate/up and QKV shapes.  achieved = 2*M*N*K / time.
Timed with CUDA events around back-to-back launches on one stream (after 3
warm-up launches); peaks from MEASURED_PEAKS.json.
"""
from __future__ import annotations

import argparse
import json
from pathlib import Path

import torch

from . import capi

ROOT = Path(__file__).resolve().parents[1]


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return j["hbm_gbs"], j["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


def _time(fn, iters):
    s = torch.cuda.current_stream()
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(iters):
        fn(i)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters  # ms per launch


def gemv_case(name, R, N, K, copies, kernel="gemv"):
    g = torch.Generator(device="cuda").manual_seed(N + K)
    Ws = [(torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16) for _ in range(copies)]
    A = torch.randn(16, K, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(R, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def fn(i):
        if kernel == "gemv_tc":
            capi.check(capi.lib().moa_k_gemv_tc(A.data_ptr(), R, Ws[i % copies].data_ptr(), N, K, out.data_ptr(), st))
        else:
            capi.check(capi.lib().moa_k_gemv(A.data_ptr(), 0, R, Ws[i % copies].data_ptr(), N, K, out.data_ptr(), st))

    ms = _time(fn, 40)
    bytes_ = 2.0 * N * K + 2.0 * R * K + 4.0 * R * N
    return {"kernel": kernel, "case": name, "rows": R, "N": N, "K": K, "us": ms * 1e3,
            "gbs": bytes_ / (ms / 1e3) / 1e9, "bytes": bytes_}


def gemm_case(name, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def fn(i):
        capi.check(capi.lib().moa_k_gemm_tc(A.data_ptr(), M, W.data_ptr(), N, K, out.data_ptr(), st))

    ms = _time(fn, 20)
    flops = 2.0 * M * N * K
    ref_ms = _time(lambda i: torch.matmul(A, W.T), 20)
    return {"kernel": "gemm_tc", "case": name, "M": M, "N": N, "K": K, "us": ms * 1e3,
            "tflops": flops / (ms / 1e3) / 1e12, "torch_matmul_tflops": flops / (ref_ms / 1e3) / 1e12}


def run():
    hbm, tf, src = peaks()
    rows = []
    for kernel in ("gemv_tc", "gemv"):
        for R in (1, 8):
            rows.append(gemv_case("1b.qkv", R, 3072, 2048, 48, kernel))
            rows.append(gemv_case("1b.gate_up", R, 16384, 2048, 16, kernel))
            rows.append(gemv_case("1b.down", R, 2048, 8192, 16, kernel))
            rows.append(gemv_case("1b.lm_head", R, 50000, 2048, 4, kernel))
            rows.append(gemv_case("8b.gate_up", R, 28672, 4096, 4, kernel))
    for M in (512, 2048):
        rows.append(gemm_case("1b.gate_up", M, 16384, 2048))
        rows.append(gemm_case("1b.qkv", M, 3072, 2048))
        rows.append(gemm_case("8b.gate_up", M, 28672, 4096))
    for r in rows:
        if "gbs" in r:
            r["frac_hbm"] = r["gbs"] / hbm
        if "tflops" in r:
            r["frac_tensor"] = r["tflops"] / tf
    return {"peaks": {"hbm_gbs": hbm, "bf16_tflops": tf, "source": src}, "cases": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--json")
    a = ap.parse_args()
    res = run()
    for r in res["cases"]:
        print(json.dumps(r))
    if a.json:
        Path(a.json).write_text(json.dumps(res, indent=1))
