// Launchers for the sm_100a kernels of the agent forward and the early-exit
// signals.  Every launcher is asynchronous on `st`.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <vector>
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

// Running softmax statistics of one vocab slice (see lm_head).
struct LmStat {
  float m;  // max logit
  float s;  // sum exp(x - m)
  float t;  // sum (x - m) exp(x - m)
  int idx;  // argmax (lowest index on ties)
};

// Device weight-row layouts (init_uniform_rows): the fused GEMV epilogues
// need RoPE pairs / gate-up pairs in adjacent output columns.
enum RowMap : int {
  kRowsIdentity = 0,
  kRowsRopeInterleave = 1,  // within each head of `hd` rows: i -> 2i (i < hd/2), 2(i-hd/2)+1
  kRowsEven = 2,            // r -> 2r     (gate rows)
  kRowsOdd = 3,             // r -> 2r + 1 (up rows)
};

// Programmatic dependent launch for the forward kernels (MOA_NO_PDL=1: off, A/B runs).
bool pdl_enabled();
// Request the maximum shared-memory carveout for a kernel (once per kernel).
void uniform_carveout(const void* fn);
// debug: per-CTA globaltimer stamps of the decode chain (stamp.cuh), nullptr = off
void forward_chain_stamp(unsigned long long* buf);
void gemv_tc_chain_stamp(unsigned long long* buf);
void gemm_tc_chain_stamp(unsigned long long* buf);
void attn_decode_chain_stamp(unsigned long long* buf);
void attn_prefill_tc_chain_stamp(unsigned long long* buf);

void init_uniform_rows(bf16* dst, long long rows, long long cols, std::uint64_t base, float scale, int map,
                       int hd, cudaStream_t st);
void fill_f32(float* dst, long long n, float v, cudaStream_t st);
// one trivial PDL kernel (measures the per-kernel cost of a launch chain)
void noop_chain_link(int* p, int ctas, cudaStream_t st);

// Tick metadata in device memory, read by every kernel of a forward so one
// captured CUDA graph per (rows, context) bucket serves every tick:
// meta[0] = live rows R, meta[1] = logits rows Rl, meta[2] = max position.
// Grids are sized for the bucket caps; CTAs past the live counts exit.
// ssq / xb (optional): per-16-column sums of squares of the rows [R][d/16]
// and their bf16 copy [R][d] (the first normed GEMV's operand)
void embed(const RowDesc* rows, int R_cap, const int* meta, const int* out_tok, const bf16* emb, int d, float* x,
           cudaStream_t st, float* ssq = nullptr, bf16* xb = nullptr);

// Fused skinny GEMM  y[r][n] = sum_k A[r][k] W[n][k]  for decode/incremental
// rows.  A is either bf16 activations or, with `norm`, the fp32 residual rows
// normalised on the fly (A = bf16(rmsnorm(x) * g), the oracle's rounding
// point).  Epilogues:
enum Epi : int { kEpiF32 = 0, kEpiResidual = 1, kEpiSwiGlu = 2, kEpiQkv = 3, kEpiLmStats = 4 };
struct LmStat;
struct GemvArgs {
  const bf16* A = nullptr;   // [R][K] bf16 (when X == nullptr)
  // Normed linear maps (RMSNorm with unit gains, applied to the fp32 product:
  // y = (bf16(x) W^T) * inv_rms(x), oracle/model.py normed_linear):
  const float* X = nullptr;  // [R][K] fp32 residual rows: operand bf16(x), inverse RMS computed in-kernel
  const float* inv = nullptr;  // or: A = bf16(x) rows and their inverse RMS [R] (prep kernel)
  float eps = 1e-5f;
  int R = 0, N = 0, K = 0;    // R: row cap (grid); live rows = meta ? meta[0] : R
  const int* meta = nullptr;
  const bf16* W = nullptr;  // [N][K] device layout
  int epi = kEpiF32;
  float* out = nullptr;      // kEpiF32: [R][N]; kEpiResidual: x [R][N] (+=)
  bf16* out_bf16 = nullptr;  // kEpiSwiGlu: a [R][N/2]; kEpiQkv: q [R][nh*hd]
  // kEpiQkv: RoPE + KV append
  const RowDesc* rows = nullptr;
  const float2* rope = nullptr;
  bf16* kpool = nullptr;
  bf16* vpool = nullptr;
  long long kv_stride = 0, layer_off = 0;
  int max_ctx = 0, nh = 0, nkv = 0, hd = 0;
  // kEpiLmStats (tensor-core LM head): greedy statistics per logits row
  LmStat* lm_part = nullptr;  // [rows][tiles]
  int* lm_cnt = nullptr;      // one int, zero-initialised once
  const int* out_idx = nullptr;
  int* out_tok = nullptr;
  float* out_lp = nullptr;
  float* out_ent = nullptr;
  float* logits = nullptr;  // optional fp32 [rows][N]
  // or (gemv_tc): A = bf16(x) rows and their per-16-column sums of squares [R][K/16]
  const float* ssq = nullptr;
  // kEpiResidual: also write the new rows' per-16-column sums of squares [R][N/16]
  // and their bf16 copy [R][N] (the next normed GEMV's operand)
  float* ssq_out = nullptr;
  bf16* xb_out = nullptr;
  // lm_head_tc with X (norm folded in): the residual rows to normalise, selected by sel[i]
  const int* sel = nullptr;
  // kEpiResidual (SIMT gemv): the residual rows were last written at least two
  // kernels back, so they are read before the PDL wait
  bool res_early = false;
  // gemv_tc / lm_head_tc: stream the weights with an L2 evict-first hint
  // (each weight byte is read once per forward; the activations, KV and
  // partials the chain re-reads keep the L2)
  bool evict_first = false;
};
void gemv(const GemvArgs& a, cudaStream_t st);  // dispatches to gemv_stream for large matrices
// HBM-streaming variant (gemv_stream.cu): persistent CTAs, cp.async.bulk ring.
bool gemv_stream_supported(const GemvArgs& a);
void gemv_stream(const GemvArgs& a, cudaStream_t st);

// ---- tensor-core prefill GEMM (gemm_tc.cu): tcgen05 + TMEM + TMA ----
// Opaque mirror of CUtensorMap (2-D bf16, K-major, SWIZZLE_128B, box 64 x rows).
struct alignas(64) TmaMap {
  unsigned char raw[128];
};
bool make_tmap_bf16(TmaMap* out, const bf16* base, long long rows, long long cols, int box_rows);
bool gemm_tc_supported(int N, int K);
// Same epilogues as gemv; A comes from map_a (bf16 rows; for a normed map
// A = bf16(x) and a.inv holds the rows' inverse RMS, applied to the products).
void gemm_tc(const TmaMap& map_a, const TmaMap& map_w, const GemvArgs& a, cudaStream_t st);
// Operand prep of a normed linear map: h[i] = bf16(x[r]) and inv[i] =
// 1 / sqrt(mean(x[r]^2) + eps), r = sel ? sel[i] : i, for i < meta[meta_idx];
// one CTA per row, 16-byte vectors.
void rmsnorm_rows(const float* x, int R_cap, const int* meta, int K, float* inv, float eps, bf16* h,
                  cudaStream_t st, const int* sel = nullptr, int meta_idx = 0);
constexpr int kTcMinRows = 17;  // ticks with more rows than the swap-AB GEMV holds use the tcgen05 GEMM (M = 128 tiles)

// ---- decode GEMV on the tensor cores, swap-AB (gemv_tc.cu) ----
// Weight map: box 64 x 128 rows (the gemm_tc weight maps); activation map:
// box 64 x 16 rows.  ws / cnt: split-K partials and per-tile counters
// (cnt zero-initialised once; the kernel leaves it zero).  Launched with
// programmatic dependent launch: weight tiles stream before the previous
// kernel has finished.
constexpr int kGemvTcRows = 16;
// ... and its wide variants (MMA N = 32 / 64) for ticks of 17..32 / 33..64 rows
// (incremental-prefill chunks: one or two 32-token chunks of a model per tick)
constexpr int kGemvTcMidRows = 32;
constexpr int kGemvTcWideRows = 64;
// rows of the activation tile (the TMA box) the swap-AB GEMV uses for R rows
constexpr int gemv_tc_box_rows(int R) { return R <= kGemvTcRows ? kGemvTcRows : R <= kGemvTcMidRows ? kGemvTcMidRows : kGemvTcWideRows; }
bool gemv_tc_supported(const GemvArgs& a);
// gemv_tc with X = fp32 residual rows normalised in-kernel (a.X, a.g, a.eps,
// a.ssq): no separate rmsnorm launch
bool gemv_tc_norm_supported(const GemvArgs& a);
int gemv_tc_splits(int N, int K, int epi);
long long gemv_tc_ws_floats(int N, int K);
void gemv_tc(const TmaMap& map_w, const TmaMap& map_x, const GemvArgs& a, float* ws, int* cnt, cudaStream_t st);
// Persistent LM head with fused greedy statistics (epi kEpiLmStats args): one
// CTA per SM over contiguous vocab tiles; part >= 16 * grid LmStat, cnt one
// int zero-initialised once.  With a.X set (and a.sel, a.g, a.eps) the CTA
// normalises the selected residual rows itself (no rmsnorm launch, no X TMA).
void lm_head_tc(const TmaMap& map_w, const TmaMap& map_x, const GemvArgs& a, LmStat* part, int* cnt, int grid,
                cudaStream_t st);  // per-CTA stamps [cta][8] (debug), nullptr = off

// o[r][h] = softmax(q k^T / sqrt(hd)) v over keys [0, pos] of the row's agent;
// keys split across CTAs (kKvSplit keys each), partials combined in split
// order by the last-arriving CTA.  `ws` >= attention_ws_floats(...) floats,
// `cnt` >= R*nh ints, zero-initialised once (the kernel leaves them zero).
constexpr int kKvSplit = 128;  // smallest split (sizes the partial workspace)
// keys per attention CTA: 8 warps x 32 for hd 64, 4 warps x 32 for hd 128
// keys per attention CTA (GQA kernel); MOA_KV_SPLIT overrides (multiple of kKvSplit)
inline int kv_split(int hd) {
  static const int env = [] {
    const char* e = std::getenv("MOA_KV_SPLIT");
    const int v = e ? std::atoi(e) : 0;
    return v >= kKvSplit && v % kKvSplit == 0 ? v : 0;
  }();
  return env ? env : (hd == 64 ? 1024 : 512);
}
long long attention_ws_floats(int R, int nh, int hd, int max_ctx);
// skip_runs: leave rows inside same-agent runs of consecutive positions to
// attention_prefill (which skips the rows alone in their run).
void attention(const bf16* q, const RowDesc* rows, int R_cap, int nsplit_cap, const int* meta, int nh, int nkv,
               int hd, const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off, int max_ctx,
               bf16* o, float* ws, int* cnt, cudaStream_t st, bool skip_runs = false);

// The same contract on TMA-staged keys (attn_decode.cu): fixed splits of
// attention_decode_tma_keys(hd) keys per CTA; kmap / vmap = the K / V pools as
// [rows][hd] TMA maps (64-row boxes, 128B swizzle).  The pools must hold
// finite values everywhere (zero-initialised): whole 64-key boxes are loaded.
int attention_decode_tma_keys(int hd);
bool attention_decode_tma_supported(int nh, int nkv, int hd, int max_ctx);
void attention_decode_tma(const TmaMap& kmap, const TmaMap& vmap, const bf16* q, const RowDesc* rows, int R_cap,
                          int nsplit_cap, const int* meta, int nh, int nkv, int hd, long long kv_stride,
                          long long layer_off, int max_ctx, bf16* o, float* ws, int* cnt, cudaStream_t st,
                          bool skip_runs = false);

// Cluster-split decode attention (attn_decode.cu): CTA = (split, kv head,
// row), the ns <= 8 splits of a row's whole 64-key boxes form a thread-block
// cluster and combine over DSMEM (no workspace); a producer warp streams each
// split's boxes through a TMA ring.  Same maps and pool contract as above.
int attention_decode_cluster_splits(int rcap, int nkv, int nbox_cap);
bool attention_decode_cluster_supported(int nh, int nkv, int hd);
void attention_decode_cluster(const TmaMap& kmap, const TmaMap& vmap, const bf16* q, const RowDesc* rows, int R_cap,
                              int ns, const int* meta, int nh, int nkv, int hd, long long kv_stride,
                              long long layer_off, int max_ctx, bf16* o, cudaStream_t st, bool skip_runs = false);

// Prefill ticks (rows of long same-agent runs): CTA = 64 consecutive rows x q
// head, keys streamed through smem once per same-agent segment; rows alone in
// their run are skipped (pair with attention(..., skip_runs = true)).  hd 64 / 128.
void attention_prefill(const bf16* q, const RowDesc* rows, int R_cap, const int* meta, int nh, int nkv, int hd,
                       const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off, int max_ctx,
                       bf16* o, cudaStream_t st);

// Prompt-prefill attention on tcgen05 (attn_prefill_tc.cu): CTA = kv head x
// 128 / hpg tick rows (M = 128 (row, q head) pairs of the GQA group), S and O
// accumulated in TMEM, K / V blocks by TMA.  qmap: make_tmap_q3d over q
// [rows][nh][hd]; kmap / vmap as for attention_decode_tma.  Rows alone in
// their run are skipped (pair with the per-row kernel, skip_runs = true).
bool make_tmap_q3d(TmaMap* out, const bf16* q, long long rows, int nh, int hd, int hpg);
// Key splits (KS <= 8): grid.z = KS CTAs per row block (one cluster), fp32
// partials through ws (attention_prefill_tc_ws_floats).
bool attention_prefill_tc_supported(int nh, int nkv, int hd);
constexpr int kPfTcMaxCtas = 2 * 148;  // key-split grids: at most two CTAs per SM
int attention_prefill_tc_splits(int R_cap, int nh, int nkv, int nblocks);
long long attention_prefill_tc_ws_floats(int hd);
void attention_prefill_tc(const TmaMap& qmap, const TmaMap& kmap, const TmaMap& vmap, const RowDesc* rows, int R_cap,
                          const int* meta, int nh, int nkv, int hd, long long kv_stride, long long layer_off,
                          int max_ctx, bf16* o, cudaStream_t st, int KS = 1, float* ws = nullptr);

// Decode ticks of small agents (every row the only row of its agent):
// RMSNorm + QKV + RoPE + KV append + attention in one launch, CTA = (row, kv
// head) with its Wqkv slabs in smem.  o as attention().
bool qkv_attention_supported(int D, int nh, int nkv, int hd);
// the fused o-projection (wo_blk != nullptr) of qkv_attention: the one check
// shared by the host (which then drops its o-projection launch) and the launcher
bool qkv_oproj_supported(int D, int nh, int nkv, int hd);
// emb / out_tok (layer 0): gather the rows' embeddings in-kernel and write X
// (the embed kernel folded in); nullptr: X holds the residual rows.  kmap /
// vmap (hd 64): the K / V pools as [rows][64] TMA maps with 64-row boxes --
// the earlier keys arrive 128B-swizzled and the attention phase runs on the
// tensor cores (mma.sync) when the whole context fits the smem stage.
// wo_blk ([nkv][D][hpg*hd], the o-projection regrouped by kv group): the
// kernel also applies x += o . Wo^T across a cluster of the row's nkv CTAs
// (DSMEM) -- the o-projection launch folded in; o is then not written.
void qkv_attention(float* X, const float* g, float eps, int D, const bf16* wqkv, const RowDesc* rows, int R_cap,
                   const int* meta, const float2* rope, int nh, int nkv, int hd, bf16* kpool, bf16* vpool,
                   long long kv_stride, long long layer_off, int max_ctx, bf16* o, cudaStream_t st,
                   const bf16* emb = nullptr, const int* out_tok = nullptr, const TmaMap* kmap = nullptr,
                   const TmaMap* vmap = nullptr, const bf16* wo_blk = nullptr);

// LM head over selected rows: logits = bf16(rmsnorm(x[sel[i]]) * g) . W^T,
// fused greedy statistics; the last CTA merges the per-slice partials and
// writes token / logprob / entropy to out_*[out_idx[i]].  `logits`
// (optional) receives the fp32 rows.  cnt: one int, zero-initialised once.
int lm_head_blocks(int V);
constexpr int kLmMaxRows = 64;
void lm_head(const float* X, const int* sel, const int* meta, const float* g, float eps, const bf16* W, int V, int d,
             LmStat* part, int* cnt, const int* out_idx, int* out_tok, float* out_lp, float* out_ent,
             float* logits, cudaStream_t st);

// ---- early-exit signals (fp64) ----
// C = exp(mean(lp[0..n))) with a sequential fp64 sum (metricq.cpp:18-23).
void ee_confidence(const float* lp, int n, double* c, cudaStream_t st);
// MockProvider rows for tokens out_tok[base .. base+n) (embedding.cpp:91-113).
void ee_mock_embed(const int* out_tok, long long base, int n, int h, std::uint64_t seed, double* emb,
                   cudaStream_t st);
// Hidden-state provider rows: emb[r][c] = x[r][c] / sqrt(mean(x[r]^2) + eps)
// (fp64) from the embedding model's fp32 final residual rows.
void ee_hidden_embed(const float* x, int n, int d, double eps, double* emb, cudaStream_t st);
// corr = correlation_from_gram(emb^T emb) (metricq.cpp:32-53), h x h.
void ee_corr(const double* emb, int n, int h, double eps, double* gram, double* corr, cudaStream_t st);
// n x n route (h > n): ahat = emb with each column scaled to unit norm (0 if
// its sum of squares <= eps); out[j] = ||ahat . stored_j^T||_F^2 for j < m
// (stored_j = stored + j * stride, d_nv[j] rows) and out[m] = ||ahat ahat^T||_F^2.
// part >= ee_cross_parts(max rows, m) doubles.
void ee_colnorm(const double* emb, int n, int h, double eps, double* ahat, cudaStream_t st);
long long ee_cross_parts(int max_n, int max_members);
void ee_cross_sumsq(const double* ahat, int n, const double* stored, const int* d_nv, int n_max_stored,
                    long long stride, int m, int h, double* part, double* out, cudaStream_t st);
// sim[j] = frob_cos_sim_corr(corr_new, corrs[j]) for j < m (metricq.cpp:55-64).
void ee_fcs(const double* corr_new, const double* corrs, int m, int h, double* sim, cudaStream_t st);
// One launch per mock-provider evaluation on the h x h route (h <= 128, m <= 16
// stored members): out[0] = C from the device logprobs, the new correlation into
// corrs[m], out[1 + k] = FCS against member k.
bool ee_fused_mock_supported(int h, int m);
void ee_fused_mock(const int* out_tok, const float* lp, long long base, int n, int h, std::uint64_t seed, double eps,
                   double* corrs, int m, double* out, cudaStream_t st);

}  // namespace moa::k
