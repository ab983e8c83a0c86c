// One agent model resident on the device: bf16 weights (hash-uniform init,
// bit-identical with oracle/model.py), the RoPE table, a KV pool for the
// agents bound to it, and the per-tick workspace.  `forward` runs one ragged
// batch of rows (decode rows + incremental-prefill rows of any agents of this
// model) through all layers and writes greedy token / logprob / entropy for
// the rows that need logits.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "../kernels/kernels.cuh"
#include "common.hpp"

namespace moa {

void cuda_check(cudaError_t e, const char* what);
#ifndef MOA_CUDA
#define MOA_CUDA(x) ::moa::cuda_check((x), #x)
#endif

struct ModelSpec {
  std::string tag;
  int d = 256, n_layers = 4, n_heads = 4, n_kv_heads = 4, head_dim = 64, ffn = 1024;
  int vocab = 50000;
  double rope_theta = 10000.0, norm_eps = 1e-5, lm_gain = 4.0;
  std::uint64_t seed = 0;

  int qkv_cols() const { return (n_heads + 2 * n_kv_heads) * head_dim; }
  long long weight_elems() const;
  double weight_bytes() const { return 2.0 * static_cast<double>(weight_elems()); }
  double decode_weight_bytes() const;  // bytes one tick must stream (all but the embedding table)
  void validate() const;
};

// Per-tick row statistics (host-computed; the probes' algorithmic bytes):
// keys = sum over rows of (pos + 1); rows alone in their same-agent run
// (decode rows) and their keys; multi-row runs' unique key prefixes
// (sum of last pos + 1) and causal (row, key) pairs.
struct TickStats {
  long long keys = 0, singles = 0, single_keys = 0, run_keys = 0, run_pairs = 0;
};

struct ForwardBuffers {
  k::RowDesc* rows = nullptr;  // [max_rows], right after sel in one allocation
  int* sel = nullptr;  // [2 * max_logit_rows + 3]: logits row index, flat output index, meta {R, Rl, max_pos}
  int sel_bytes = 0;   // sel region padded to 16 bytes (rows start there)
};

// Per-kernel CUDA-event probes (bench roofline): when attached, forwards run
// without graphs and every launch is bracketed by an event pair together with
// its algorithmic bytes.
struct KernelProbes {
  // decode-regime kinds (rows <= 16: swap-AB GEMVs, per-row attention, the
  // fused small-agent kernel) and prefill-regime kinds (tcgen05 GEMM, tiled
  // prompt attention) are kept apart: they have different rooflines
  enum Kind {
    Embed = 0, Qkv, AttnDecode, OProj, GateUp, Down, LmHead, QkvAttn, AttnPrefill, PfQkv, PfOProj, PfGateUp, PfDown,
    kKinds
  };
  struct Rec {
    int kind;
    double bytes, flops;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  std::size_t next = 0;
  std::vector<Rec> recs;
  cudaEvent_t event();
  void begin(int kind, double bytes, cudaStream_t st, double flops = 0.0);
  void end(cudaStream_t st);
  void reset() {
    next = 0;
    recs.clear();
  }
  ~KernelProbes();
};

class DeviceModel {
 public:
  void attach_probes(KernelProbes* p) { probes_ = p; }
  void set_tensor_cores(bool on) { use_tc_ = on; }
  bool tensor_cores_ready() const { return tc_ok_; }
  DeviceModel(const ModelSpec& spec, int max_agents, int max_ctx, int max_rows, int max_logit_rows,
              cudaStream_t st, bool use_graphs = true);
  ~DeviceModel();
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;

  const ModelSpec& spec() const { return spec_; }
  int bind_agent();  // next free KV slot
  void reset_bindings() { bound_ = 0; }
  int max_rows() const { return max_rows_; }
  int max_logit_rows() const { return max_lrows_; }
  const ForwardBuffers& buffers() const { return buf_; }
  // Two tick-metadata blobs: the next tick's upload lands in one while the
  // current tick's graph reads the other (graphs are keyed by the blob).
  void use_blob(int b);
  int blob() const { return blob_; }
  // Decode runs: K consecutive pure-decode ticks launched as one graph, each
  // tick reading its own compact metadata blob (run area [2][kMaxRun][stride],
  // rows <= max_logit_rows).  run_blob(p) = device base of parity p.
  static constexpr int kMaxRun = 8;
  std::size_t run_stride() const { return run_stride_; }
  void* run_blob(int parity) const { return static_cast<char*>(run_area_) + parity * kMaxRun * run_stride_; }
  bool runs_supported() const { return use_graphs_ && !probes_; }
  const float* residual() const { return x_; }  // final residual rows of the last forward

  // R rows / Rl logits rows already resident in buffers(); out_* are the
  // engine's flat per-agent output arrays; logits (optional) [Rl][V] fp32.
  // distinct: every row belongs to a different agent (a pure decode tick)
  // prefill: the rows are long same-agent runs (prompt prefill): tiled attention
  // (singles: some rows are alone in their run -- the per-row kernel serves them)
  void forward(int R, int Rl, int max_pos, const TickStats& ts, const int* out_tok_read, int* out_tok, float* out_lp,
               float* out_ent, float* logits, cudaStream_t st, bool distinct = false, bool prefill = false,
               bool singles = true);
  // K ticks of R decode rows each (every row its own agent, one logits row per
  // row), metadata already in run_blob(parity); max_pos of the last tick.
  void forward_run(int K, int R, int max_pos, const int* out_tok_read, int* out_tok, float* out_lp, float* out_ent,
                   cudaStream_t st, int parity);

  // Algorithmic bytes one forward must move for weights (every tick reads the
  // full weight set once) -- the roofline basis.
  double weight_bytes() const { return spec_.decode_weight_bytes(); }
  int graphs() const { return static_cast<int>(graphs_.size()); }

 private:
  void launch(int rcap, int nsplit, bool with_logits, const int* out_tok_read, int* out_tok, float* out_lp,
              float* out_ent, float* logits, cudaStream_t st, bool distinct, bool prefill = false,
              bool singles = true);
  bool qkv_attn_ok_ = false, use_qkv_attn_ = true;  // fused QKV + attention for small-agent decode ticks
  bool use_prefill_attn_ = true;  // tiled prefill attention for prompt-prefill ticks (MOA_PREFILL_ATTN)
  std::map<std::tuple<int, int, int, int>, cudaGraphExec_t> graphs_;
  ModelSpec spec_;
  int max_agents_, max_ctx_, max_rows_, max_lrows_;
  bool use_graphs_ = true;
  bool use_tc_ = true;  // tensor-core path for ticks with >= kTcMinRows rows
  bool tc_ok_ = false;
  // RMSNorm folded into the swap-AB decode GEMVs (qkv, gate/up): operand
  // bf16(x) in hn_, inverse RMS from the 16-column sums of squares ssq_
  bool nfold_ok_ = false, use_nfold_ = true;
  float* ssq_ = nullptr;
  float* inv_ = nullptr;  // prep launches: the rows' inverse RMS [max_rows]
  int lm_grid_ = 148;  // persistent LM head: one CTA per SM
  // decode GEMVs stream their weights with an L2 evict-first hint
  // (MOA_EVICT_FIRST=0: off; measured -3.5..-6% per 1B / 8B decode tick)
  bool evict_first_ = true;
  void graphs_clear();
  struct LayerMaps {
    k::TmaMap wqkv, wo, wgu, wd;
  };
  std::vector<LayerMaps> wmaps_;
  k::TmaMap wmap_lm_;  // LM head [V][d], 128-row boxes
  k::TmaMap kmap_, vmap_;  // K / V pools as [rows][hd], 64-row boxes (fused QKV + attention, hd 64)
  k::bf16* wo_blk_ = nullptr;  // [L][nkv][D][hpg*hd]: Wo regrouped for the fused o-projection
  bool kv_maps_ok_ = false;
  k::TmaMap qmap3_;     // q [rows][nh][hd] as a 3-D map (GQA-group boxes) for the tcgen05 prefill attention
  bool pf_tc_ = false;  // prompt-prefill attention on tcgen05 (attn_prefill_tc.cu)
  bool attn_tma_ = false;  // decode rows: TMA-staged attention (attn_decode.cu)
  bool attn_cluster_ = false;  // decode rows: cluster-split TMA-ring attention (attn_decode.cu, default)
  int split_keys_ = 512;   // keys per attention CTA (sizes the graphs' split buckets)
  k::TmaMap map_hn_, map_h_attn_, map_h_ffn_;        // A operands, 128-row boxes (prefill)
  k::TmaMap map_hn16_, map_h_attn16_, map_h_ffn16_;  // 16-row boxes (decode, swap-AB)
  k::TmaMap map_hn32_, map_h_attn32_, map_h_ffn32_;  // 32-row boxes (its wide variants)
  k::TmaMap map_hn64_, map_h_attn64_, map_h_ffn64_;  // 64-row boxes
  float* pf_ws_ = nullptr;  // key-split partials of the tcgen05 prefill attention
  float* gv_ws_ = nullptr;                           // gemv_tc split-K partials
  int* gv_cnt_ = nullptr;
  k::bf16* hn_ = nullptr;                      // normalised rows for the tensor-core path
  KernelProbes* probes_ = nullptr;
  int live_R_ = 0, live_Rl_ = 0;
  TickStats live_;
  int bound_ = 0;
  // weights
  k::bf16* wbase_ = nullptr;
  k::bf16* emb_ = nullptr;
  k::bf16* lm_ = nullptr;
  struct Layer {
    k::bf16 *wqkv, *wo, *wgu, *wd;
  };
  std::vector<Layer> layers_;
  float* ones_ = nullptr;  // RMSNorm gains (all 1.0)
  float2* rope_ = nullptr;
  // KV pools [agents][L][nkv][max_ctx][hd]
  k::bf16* kpool_ = nullptr;
  k::bf16* vpool_ = nullptr;
  long long kv_stride_ = 0, layer_stride_ = 0;
  // workspace
  float* x_ = nullptr;
  k::bf16* h_ = nullptr;
  k::bf16* q_ = nullptr;
  float* attn_ws_ = nullptr;
  long long attn_ws_floats_ = 0;
  int* attn_cnt_ = nullptr;
  k::LmStat* part_ = nullptr;
  int* lm_cnt_ = nullptr;
  ForwardBuffers buf_;
  void* meta_blob_ = nullptr;  // [2][sel_bytes + rows]
  void* run_area_ = nullptr;   // [2][kMaxRun][run_stride_]
  std::size_t run_stride_ = 0;
  std::size_t blob_bytes_ = 0;
  int blob_ = 0;
};

}  // namespace moa
