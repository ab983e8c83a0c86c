// Launchers for the sm_100a kernels of the agent forward and the early-exit
// signals.  Every launcher is asynchronous on `st`.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace moa::k {

using bf16 = __nv_bfloat16;

// One ragged-batch row of a tick: the agent's KV slot inside its model's
// pool, the absolute position, the input token (>= 0 literal, < 0 symbolic:
// out_tok[-1 - tok]) and the flat output index (-1: no logits for this row).
struct RowDesc {
  int kv;
  int pos;
  int tok;
  int out;
};

// Running softmax statistics of one vocab slice (see lm_head_stats).
struct LmStat {
  float m;    // max logit
  float s;    // sum exp(x - m)
  float t;    // sum (x - m) exp(x - m)
  int idx;    // argmax (lowest index on ties)
};

void init_uniform(bf16* dst, long long n, std::uint64_t base, float scale, cudaStream_t st);
void fill_f32(float* dst, long long n, float v, cudaStream_t st);

void embed(const RowDesc* rows, int R, const int* out_tok, const bf16* emb, int d, float* x,
           cudaStream_t st);
// h[i] = bf16(rmsnorm(x[sel ? sel[i] : i]) * g)
void rmsnorm(const float* x, const int* sel, int R, int d, const float* g, float eps, bf16* h,
             cudaStream_t st);
// P[s][r][n] = sum_{k in slice s} A[r][k] * W[n][k]   (A bf16 [R][K], W bf16 [N][K])
void gemm_skinny(const bf16* A, int R, const bf16* W, int N, int K, int S, float* P,
                 cudaStream_t st);
// x[r][n] += sum_s P[s][r][n]
void residual_add(float* x, const float* P, int S, int R, int N, cudaStream_t st);
// a[r][j] = bf16(silu(g) * u), g/u = sum_s P[s][r][j], P[s][r][ffn + j]
void swiglu(const float* P, int S, int R, int ffn, bf16* a, cudaStream_t st);
// RoPE + KV append: q -> bf16 q buffer, k/v -> the agent's cache at `pos`.
void rope_kv(const float* P, int S, const RowDesc* rows, int R, int nh, int nkv, int hd,
             const float2* rope, bf16* q, bf16* kpool, bf16* vpool, long long kv_stride,
             long long layer_off, int max_ctx, cudaStream_t st);
// o[r][h] = softmax(q k^T / sqrt(hd)) v over keys [0, pos] of the row's agent.
void attention(const bf16* q, const RowDesc* rows, int R, int nh, int nkv, int hd,
               const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off,
               int max_ctx, bf16* o, cudaStream_t st);
// Fused LM head + greedy statistics over the selected rows: per-block partial
// (max, sum e^, sum (x-m) e^, argmax); `logits` (optional) receives fp32 rows.
int lm_head_blocks(int V);
void lm_head_stats(const bf16* h, int Rl, const bf16* W, int V, int d, LmStat* part,
                   float* logits, cudaStream_t st);
// Merge partials and write token / logprob / entropy at out[]; out index per row.
void lm_merge(const LmStat* part, int Rl, int nblk, const int* out_idx, int* out_tok,
              float* out_lp, float* out_ent, cudaStream_t st);

// ---- early-exit signals (fp64) ----
// C = exp(mean(lp[0..n))) with a sequential fp64 sum (metricq.cpp:18-23).
void ee_confidence(const float* lp, int n, double* c, cudaStream_t st);
// MockProvider rows for tokens out_tok[base .. base+n) (embedding.cpp:91-113).
void ee_mock_embed(const int* out_tok, long long base, int n, int h, std::uint64_t seed, double* emb,
                   cudaStream_t st);
// corr = correlation_from_gram(emb^T emb) (metricq.cpp:32-53), h x h.
void ee_corr(const double* emb, int n, int h, double eps, double* gram, double* corr,
             cudaStream_t st);
// sim[j] = frob_cos_sim_corr(corr_new, corrs[j]) for j < m (metricq.cpp:55-64).
void ee_fcs(const double* corr_new, const double* corrs, int m, int h, double* sim,
            cudaStream_t st);

}  // namespace moa::k
