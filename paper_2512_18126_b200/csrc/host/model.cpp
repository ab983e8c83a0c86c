#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace moa {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

long long ModelSpec::weight_elems() const {
  const long long D = d, hd = head_dim;
  long long per_layer = qkv_cols() * D + D * n_heads * hd + 2LL * ffn * D + D * ffn;
  return 2LL * vocab * D + n_layers * per_layer;
}

double ModelSpec::decode_weight_bytes() const {
  // every tick reads all layer weights and the LM head; the embedding table
  // is gathered row-wise (R rows), so it is not part of the per-tick stream
  const long long D = d;
  return 2.0 * static_cast<double>(weight_elems() - static_cast<long long>(vocab) * D);
}

void ModelSpec::validate() const {
  if (d <= 0 || n_layers <= 0 || n_heads <= 0 || n_kv_heads <= 0 || ffn <= 0 || vocab <= 0)
    throw ValidationError("model " + tag + ": dimensions must be positive");
  if (head_dim != 64 && head_dim != 128) throw ValidationError("model " + tag + ": head_dim must be 64 or 128");
  if (n_heads % n_kv_heads) throw ValidationError("model " + tag + ": n_heads % n_kv_heads != 0");
  if (n_heads / n_kv_heads > 4) throw ValidationError("model " + tag + ": at most 4 query heads per kv head");
  for (int k : {d, n_heads * head_dim, ffn})
    if (k % 256) throw ValidationError("model " + tag + ": GEMM K dims must be multiples of 256");
}

namespace {

// base_T = hash_combine(hash_combine(seed, fnv1a(tag)), fnv1a(T)); see oracle/model.py
std::uint64_t tensor_base(const ModelSpec& s, const std::string& name) {
  return rng::hash_combine(rng::hash_combine(s.seed, rng::fnv1a(s.tag)), rng::fnv1a(name));
}

float tensor_scale(const ModelSpec& s, const std::string& name, int k_in) {
  if (name == "emb") return 1.0f;
  if (name == "lm") return static_cast<float>(std::sqrt(3.0 / s.d) * s.lm_gain);
  return static_cast<float>(std::sqrt(3.0 / k_in));
}

template <class T>
void dev_alloc(T** p, long long n) {
  MOA_CUDA(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * static_cast<std::size_t>(n)));
}

}  // namespace

DeviceModel::DeviceModel(const ModelSpec& spec, int max_agents, int max_ctx, int max_rows, int max_logit_rows,
                         cudaStream_t st, bool use_graphs)
    : spec_(spec), max_agents_(max_agents), max_ctx_(max_ctx), max_rows_(max_rows), max_lrows_(max_logit_rows),
      use_graphs_(use_graphs) {
  spec_.validate();
  if (max_ctx > 8192) throw ValidationError("model " + spec.tag + ": max_ctx above 8192 is not supported");
  const ModelSpec& s = spec_;
  const long long D = s.d, hd = s.head_dim, V = s.vocab;
  dev_alloc(&wbase_, s.weight_elems());
  k::bf16* p = wbase_;
  auto take = [&](long long n) {
    k::bf16* r = p;
    p += n;
    return r;
  };
  // Logical tensors (oracle/model.py names) written into the device layout:
  // q/k rows interleave RoPE pairs, gate/up rows interleave (gemv epilogues).
  auto init = [&](k::bf16* dst, const std::string& name, long long rows, long long cols, int map) {
    k::init_uniform_rows(dst, rows, cols, tensor_base(s, name), tensor_scale(s, name, static_cast<int>(cols)), map,
                         s.head_dim, st);
  };
  emb_ = take(V * D);
  init(emb_, "emb", V, D, k::kRowsIdentity);
  for (int l = 0; l < s.n_layers; ++l) {
    Layer L{};
    const std::string pre = "L" + std::to_string(l) + ".";
    L.wqkv = take(s.qkv_cols() * D);
    init(L.wqkv, pre + "wq", s.n_heads * hd, D, k::kRowsRopeInterleave);
    init(L.wqkv + s.n_heads * hd * D, pre + "wk", s.n_kv_heads * hd, D, k::kRowsRopeInterleave);
    init(L.wqkv + (s.n_heads + s.n_kv_heads) * hd * D, pre + "wv", s.n_kv_heads * hd, D, k::kRowsIdentity);
    L.wo = take(D * s.n_heads * hd);
    init(L.wo, pre + "wo", D, s.n_heads * hd, k::kRowsIdentity);
    L.wgu = take(2LL * s.ffn * D);
    init(L.wgu, pre + "wg", s.ffn, D, k::kRowsEven);
    init(L.wgu, pre + "wu", s.ffn, D, k::kRowsOdd);
    L.wd = take(D * s.ffn);
    init(L.wd, pre + "wd", D, s.ffn, k::kRowsIdentity);
    layers_.push_back(L);
  }
  lm_ = take(V * D);
  init(lm_, "lm", V, D, k::kRowsIdentity);
  if (const char* f = std::getenv("MOA_EVICT_FIRST")) evict_first_ = f[0] != '0';

  const int maxd = std::max({s.d, s.ffn, s.n_heads * s.head_dim});
  dev_alloc(&ones_, maxd);
  k::fill_f32(ones_, maxd, 1.0f, st);

  // RoPE table in fp64 libm then one cast (identical to oracle/model.py rope_table)
  const int half = s.head_dim / 2;
  std::vector<float2> tab(static_cast<std::size_t>(max_ctx) * half);
  for (int pos = 0; pos < max_ctx; ++pos)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(s.rope_theta, -2.0 * i / s.head_dim);
      const double a = pos * inv;
      tab[static_cast<std::size_t>(pos) * half + i] =
          make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
    }
  dev_alloc(&rope_, static_cast<long long>(tab.size()));
  MOA_CUDA(cudaMemcpyAsync(rope_, tab.data(), sizeof(float2) * tab.size(), cudaMemcpyHostToDevice, st));

  layer_stride_ = static_cast<long long>(s.n_kv_heads) * max_ctx * hd;
  kv_stride_ = layer_stride_ * s.n_layers;
  dev_alloc(&kpool_, kv_stride_ * max_agents);
  dev_alloc(&vpool_, kv_stride_ * max_agents);
  // finite everywhere: the TMA decode attention stages whole 64-key boxes
  // (keys past a row's position are masked, but 0 * NaN would not be)
  MOA_CUDA(cudaMemsetAsync(kpool_, 0, sizeof(k::bf16) * kv_stride_ * max_agents, st));
  MOA_CUDA(cudaMemsetAsync(vpool_, 0, sizeof(k::bf16) * kv_stride_ * max_agents, st));

  dev_alloc(&x_, static_cast<long long>(max_rows) * D);
  dev_alloc(&h_, static_cast<long long>(max_rows) * maxd);
  dev_alloc(&q_, static_cast<long long>(max_rows) * s.n_heads * hd);
  attn_ws_floats_ = k::attention_ws_floats(max_rows, s.n_heads, s.head_dim, max_ctx);
  dev_alloc(&attn_ws_, attn_ws_floats_);
  dev_alloc(&attn_cnt_, static_cast<long long>(max_rows) * s.n_heads);
  MOA_CUDA(cudaMemsetAsync(attn_cnt_, 0, sizeof(int) * max_rows * s.n_heads, st));
  {
    int dev = 0;
    MOA_CUDA(cudaGetDevice(&dev));
    MOA_CUDA(cudaDeviceGetAttribute(&lm_grid_, cudaDevAttrMultiProcessorCount, dev));
  }
  dev_alloc(&part_, std::max<long long>(static_cast<long long>(max_logit_rows) * k::lm_head_blocks(s.vocab),
                                        static_cast<long long>(k::kGemvTcRows) * lm_grid_));
  dev_alloc(&lm_cnt_, 1);
  MOA_CUDA(cudaMemsetAsync(lm_cnt_, 0, sizeof(int), st));
  // tick metadata in one allocation, uploaded with one copy per tick:
  // [sel: lsel (L) | lout (L) | meta (3)] padded to 16 bytes, then the rows
  buf_.sel_bytes = static_cast<int>(((2LL * max_logit_rows + 3) * sizeof(int) + 15) / 16 * 16);
  blob_bytes_ = (buf_.sel_bytes + sizeof(k::RowDesc) * static_cast<std::size_t>(max_rows) + 255) / 256 * 256;
  MOA_CUDA(cudaMalloc(&meta_blob_, 2 * blob_bytes_));
  use_blob(0);
  run_stride_ = (buf_.sel_bytes + sizeof(k::RowDesc) * static_cast<std::size_t>(max_logit_rows) + 255) / 256 * 256;
  MOA_CUDA(cudaMalloc(&run_area_, 2 * kMaxRun * run_stride_));
  dev_alloc(&hn_, static_cast<long long>(max_rows) * D);
  // TMA descriptors for the tensor-core prefill path (weights: 128-row boxes)
  tc_ok_ = k::gemm_tc_supported(s.qkv_cols(), D) && k::gemm_tc_supported(D, s.n_heads * s.head_dim) &&
           k::gemm_tc_supported(2 * s.ffn, D) && k::gemm_tc_supported(D, s.ffn);
  for (const Layer& L : layers_) {
    LayerMaps m{};
    tc_ok_ = tc_ok_ && k::make_tmap_bf16(&m.wqkv, L.wqkv, s.qkv_cols(), D, 128) &&
             k::make_tmap_bf16(&m.wo, L.wo, D, static_cast<long long>(s.n_heads) * hd, 128) &&
             k::make_tmap_bf16(&m.wgu, L.wgu, 2LL * s.ffn, D, 128) && k::make_tmap_bf16(&m.wd, L.wd, D, s.ffn, 128);
    wmaps_.push_back(m);
  }
  tc_ok_ = tc_ok_ && k::make_tmap_bf16(&wmap_lm_, lm_, V, D, 128) && k::make_tmap_bf16(&map_hn_, hn_, max_rows, D, 128) &&
           k::make_tmap_bf16(&map_h_attn_, h_, max_rows, static_cast<long long>(s.n_heads) * hd, 128) &&
           k::make_tmap_bf16(&map_h_ffn_, h_, max_rows, s.ffn, 128) &&
           k::make_tmap_bf16(&map_hn16_, hn_, max_rows, D, k::kGemvTcRows) &&
           k::make_tmap_bf16(&map_h_attn16_, h_, max_rows, static_cast<long long>(s.n_heads) * hd, k::kGemvTcRows) &&
           k::make_tmap_bf16(&map_h_ffn16_, h_, max_rows, s.ffn, k::kGemvTcRows) &&
           k::make_tmap_bf16(&map_hn32_, hn_, max_rows, D, k::kGemvTcMidRows) &&
           k::make_tmap_bf16(&map_h_attn32_, h_, max_rows, static_cast<long long>(s.n_heads) * hd, k::kGemvTcMidRows) &&
           k::make_tmap_bf16(&map_h_ffn32_, h_, max_rows, s.ffn, k::kGemvTcMidRows) &&
           k::make_tmap_bf16(&map_hn64_, hn_, max_rows, D, k::kGemvTcWideRows) &&
           k::make_tmap_bf16(&map_h_attn64_, h_, max_rows, static_cast<long long>(s.n_heads) * hd, k::kGemvTcWideRows) &&
           k::make_tmap_bf16(&map_h_ffn64_, h_, max_rows, s.ffn, k::kGemvTcWideRows);
  long long ws = 0;
  for (auto [n, kk] : {std::pair<int, int>{s.qkv_cols(), s.d}, {s.d, s.n_heads * s.head_dim}, {2 * s.ffn, s.d},
                       {s.d, s.ffn}})
    ws = std::max(ws, k::gemv_tc_ws_floats(n, kk));
  dev_alloc(&gv_ws_, ws);
  dev_alloc(&gv_cnt_, (std::max({s.qkv_cols(), 2 * s.ffn, s.d}) + 127) / 128);
  qkv_attn_ok_ = k::qkv_attention_supported(D, s.n_heads, s.n_kv_heads, static_cast<int>(hd));
  {
    // the o-projection regrouped by kv group, [L][nkv][D][hpg*hd], for the fused
    // QKV + attention + o-projection decode kernel (small agents; MOA_FUSE_O=0: off)
    const char* e = std::getenv("MOA_FUSE_O");
    const int hpg = s.n_heads / s.n_kv_heads;
    const long long blk = static_cast<long long>(D) * hpg * hd;
    if (qkv_attn_ok_ && !(e && e[0] == '0') && k::qkv_oproj_supported(D, s.n_heads, s.n_kv_heads, static_cast<int>(hd))) {
      dev_alloc(&wo_blk_, blk * s.n_kv_heads * s.n_layers);
      for (int l = 0; l < s.n_layers; ++l)
        for (int gq = 0; gq < s.n_kv_heads; ++gq)
          MOA_CUDA(cudaMemcpy2DAsync(wo_blk_ + (static_cast<long long>(l) * s.n_kv_heads + gq) * blk, hpg * hd * 2,
                                     layers_[static_cast<std::size_t>(l)].wo + static_cast<long long>(gq) * hpg * hd,
                                     static_cast<long long>(s.n_heads) * hd * 2, hpg * hd * 2, D,
                                     cudaMemcpyDeviceToDevice, st));
    }
  }
  // K / V pools as [rows][hd] TMA maps (64-key boxes) for the fused kernel's swizzled key stage
  kv_maps_ok_ = k::make_tmap_bf16(&kmap_, kpool_, kv_stride_ * max_agents / hd, hd, 64) &&
                k::make_tmap_bf16(&vmap_, vpool_, kv_stride_ * max_agents / hd, hd, 64);
  // decode rows of GQA agents: TMA-staged attention (MOA_DECODE_TMA=0: the register-staged kernel)
  attn_tma_ = kv_maps_ok_ && k::attention_decode_tma_supported(s.n_heads, s.n_kv_heads, static_cast<int>(hd), max_ctx);
  if (const char* e = std::getenv("MOA_DECODE_TMA")) attn_tma_ = attn_tma_ && e[0] != '0';
  // prompt-prefill ticks: the tcgen05 attention (MOA_PREFILL_TC=0: the mma.sync kernel)
  pf_tc_ = kv_maps_ok_ && k::attention_prefill_tc_supported(s.n_heads, s.n_kv_heads, static_cast<int>(hd)) &&
           k::make_tmap_q3d(&qmap3_, q_, max_rows, s.n_heads, static_cast<int>(hd), s.n_heads / s.n_kv_heads);
  if (const char* e = std::getenv("MOA_PREFILL_TC")) pf_tc_ = pf_tc_ && e[0] != '0';
  if (pf_tc_) {  // key-split partials of the prefill attention (chunk ticks)
    dev_alloc(&pf_ws_, k::attention_prefill_tc_ws_floats(static_cast<int>(hd)));
  }
  // default: the cluster-split kernel (MOA_DECODE_CLUSTER=0: the fixed-split TMA kernel)
  attn_cluster_ = kv_maps_ok_ && k::attention_decode_cluster_supported(s.n_heads, s.n_kv_heads, static_cast<int>(hd));
  if (const char* e = std::getenv("MOA_DECODE_CLUSTER")) attn_cluster_ = attn_cluster_ && e[0] != '0';
  split_keys_ = attn_cluster_ ? 64
                : attn_tma_   ? k::attention_decode_tma_keys(static_cast<int>(hd))
                              : k::kv_split(static_cast<int>(hd));
  if (const char* e = std::getenv("MOA_QKV_ATTN")) use_qkv_attn_ = std::string(e) != "0";
  if (const char* e = std::getenv("MOA_PREFILL_ATTN")) use_prefill_attn_ = std::string(e) != "0";
  // RMSNorm folded into the decode GEMVs: ssq partials [16 rows][d/16]
  dev_alloc(&ssq_, static_cast<long long>(k::kGemvTcWideRows) * (D / 16));
  dev_alloc(&inv_, static_cast<long long>(max_rows));
  {
    k::GemvArgs q1, g1, o1, d1;
    q1.R = g1.R = o1.R = d1.R = k::kGemvTcRows;
    q1.N = s.qkv_cols(), q1.K = D, g1.N = 2 * s.ffn, g1.K = D;
    o1.N = D, o1.K = s.n_heads * s.head_dim, d1.N = D, d1.K = s.ffn;
    q1.ssq = g1.ssq = ssq_;
    q1.epi = k::kEpiQkv, g1.epi = k::kEpiSwiGlu;
    o1.epi = d1.epi = k::kEpiResidual;
    nfold_ok_ = tc_ok_ && D % 16 == 0 && k::gemv_tc_norm_supported(q1) && k::gemv_tc_norm_supported(g1) &&
                k::gemv_tc_supported(o1) && k::gemv_tc_supported(d1);
    // Decode ticks: the residual GEMVs (and the embedding gather) write x, its
    // bf16 copy (the next normed GEMV's TMA operand) and 16-column sums of
    // squares; the normed GEMVs compute the rows' inverse RMS from those while
    // their weights stream -- no RMSNorm launch and no staging on the critical
    // path.  MOA_NORM_FOLD=0: a prep launch per normed GEMV instead.
    use_nfold_ = true;
    if (const char* e = std::getenv("MOA_NORM_FOLD")) use_nfold_ = std::string(e) != "0";
  }
  MOA_CUDA(cudaMemsetAsync(gv_cnt_, 0, sizeof(int) * ((std::max({s.qkv_cols(), 2 * s.ffn, s.d}) + 127) / 128), st));
  MOA_CUDA(cudaGetLastError());
}

void DeviceModel::use_blob(int b) {
  blob_ = b & 1;
  char* base = static_cast<char*>(meta_blob_) + blob_ * blob_bytes_;
  buf_.sel = reinterpret_cast<int*>(base);
  buf_.rows = reinterpret_cast<k::RowDesc*>(base + buf_.sel_bytes);
}

DeviceModel::~DeviceModel() {
  for (auto& [key, exec] : graphs_) cudaGraphExecDestroy(exec);
  for (void* ptr : {static_cast<void*>(wbase_), static_cast<void*>(ones_), static_cast<void*>(rope_),
                    static_cast<void*>(kpool_), static_cast<void*>(vpool_), static_cast<void*>(x_),
                    static_cast<void*>(h_), static_cast<void*>(q_), static_cast<void*>(attn_ws_),
                    static_cast<void*>(attn_cnt_), static_cast<void*>(part_), static_cast<void*>(lm_cnt_),
                    meta_blob_, run_area_, static_cast<void*>(hn_), static_cast<void*>(wo_blk_),
                    static_cast<void*>(gv_ws_), static_cast<void*>(gv_cnt_), static_cast<void*>(ssq_),
                    static_cast<void*>(inv_), static_cast<void*>(pf_ws_)})
    if (ptr) cudaFree(ptr);
}

int DeviceModel::bind_agent() {
  if (bound_ >= max_agents_)
    throw ValidationError("model " + spec_.tag + ": agent capacity " + std::to_string(max_agents_) + " exhausted");
  return bound_++;
}

cudaEvent_t KernelProbes::event() {
  if (next == pool.size()) {
    cudaEvent_t e;
    MOA_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[next++];
}

void KernelProbes::begin(int kind, double bytes, cudaStream_t st, double flops) {
  Rec r{kind, bytes, flops, event(), event()};
  MOA_CUDA(cudaEventRecord(r.a, st));
  recs.push_back(r);
}

void KernelProbes::end(cudaStream_t st) { MOA_CUDA(cudaEventRecord(recs.back().b, st)); }

KernelProbes::~KernelProbes() {
  for (auto e : pool) cudaEventDestroy(e);
}

namespace {
// Smallest row-count bucket a tick graph is captured for (MOA_RCAP_MIN):
// exact power-of-two buckets keep the decode attention's grid (rows x kv
// heads x splits) free of dead CTAs, whose late scheduling would hold back
// the dependent launch of the o-projection (measured: -1.3 us per 8B layer).
int rcap_min() {
  static const int v = [] {
    const char* e = std::getenv("MOA_RCAP_MIN");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  return v;
}

int pow2_at_least(int v, int lo) {
  int p = lo;
  while (p < v) p <<= 1;
  return p;
}
}  // namespace

void DeviceModel::forward(int R, int Rl, int max_pos, const TickStats& ts, const int* out_tok_read, int* out_tok,
                          float* out_lp, float* out_ent, float* logits, cudaStream_t st, bool distinct, bool prefill,
                          bool singles) {
  // (tensor-core ticks only: the GEMV-only path keeps every row's attention in
  // one kernel, so its tokens stay bit-identical across schedule modes)
  prefill = prefill && use_prefill_attn_ && use_tc_;
  if (R <= 0) return;
  if (R > max_rows_) throw RunError("model " + spec_.tag + ": tick rows exceed workspace");
  if (Rl > max_lrows_ || Rl > k::kLmMaxRows) throw RunError("model " + spec_.tag + ": logits rows exceed workspace");
  if (max_pos >= max_ctx_) throw RunError("model " + spec_.tag + ": position exceeds max_ctx");
  // bucket caps: one graph serves every tick whose live counts fit them
  const int rcap = std::min(pow2_at_least(R, rcap_min()), max_rows_);
  const int ks = split_keys_;
  const int nsplit = pow2_at_least((max_pos + ks) / ks, 1);
  if (!use_graphs_ || probes_) {
    live_R_ = R;
    live_Rl_ = Rl;
    live_ = ts;
    launch(rcap, nsplit, Rl > 0, out_tok_read, out_tok, out_lp, out_ent, logits, st, distinct, prefill, singles);
    return;
  }
  const auto key = std::make_tuple(rcap, nsplit, (Rl > 0 ? 1 : 0) | (use_tc_ ? 2 : 0) |
                                                     (distinct ? 8 : 0) | (blob_ << 4) | (prefill ? 32 : 0) |
                                                     (prefill && !singles ? 64 : 0),
                                   logits ? 1 : 0);
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    cudaGraph_t g = nullptr;
    MOA_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    launch(rcap, nsplit, Rl > 0, out_tok_read, out_tok, out_lp, out_ent, logits, st, distinct, prefill, singles);
    MOA_CUDA(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t exec = nullptr;
    MOA_CUDA(cudaGraphInstantiate(&exec, g, 0));
    MOA_CUDA(cudaGraphDestroy(g));
    it = graphs_.emplace(key, exec).first;
  }
  MOA_CUDA(cudaGraphLaunch(it->second, st));
}

void DeviceModel::forward_run(int K, int R, int max_pos, const int* out_tok_read, int* out_tok, float* out_lp,
                              float* out_ent, cudaStream_t st, int parity) {
  if (K < 2 || K > kMaxRun || !runs_supported()) throw RunError("model " + spec_.tag + ": invalid decode run");
  if (R <= 0 || R > max_lrows_ || R > k::kLmMaxRows) throw RunError("model " + spec_.tag + ": run rows exceed workspace");
  if (max_pos >= max_ctx_) throw RunError("model " + spec_.tag + ": position exceeds max_ctx");
  const int rcap = std::min(pow2_at_least(R, rcap_min()), max_rows_);
  const int ks = split_keys_;
  const int nsplit = pow2_at_least((max_pos + ks) / ks, 1);  // the last tick's: a cap for the earlier ones
  const auto key = std::make_tuple(rcap, nsplit, 1 | (use_tc_ ? 2 : 0) | 8 | (parity << 4),
                                   2 * K);
  auto it = graphs_.find(key);
  if (it == graphs_.end()) {
    const int keep = blob_;
    cudaGraph_t g = nullptr;
    MOA_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < K; ++j) {
      char* base = static_cast<char*>(run_blob(parity)) + j * run_stride_;
      buf_.sel = reinterpret_cast<int*>(base);
      buf_.rows = reinterpret_cast<k::RowDesc*>(base + buf_.sel_bytes);
      launch(rcap, nsplit, true, out_tok_read, out_tok, out_lp, out_ent, nullptr, st, true);
    }
    MOA_CUDA(cudaStreamEndCapture(st, &g));
    use_blob(keep);
    cudaGraphExec_t exec = nullptr;
    MOA_CUDA(cudaGraphInstantiate(&exec, g, 0));
    MOA_CUDA(cudaGraphDestroy(g));
    it = graphs_.emplace(key, exec).first;
  }
  MOA_CUDA(cudaGraphLaunch(it->second, st));
}

void DeviceModel::launch(int rcap, int nsplit, bool with_logits, const int* out_tok_read, int* out_tok,
                         float* out_lp, float* out_ent, float* logits, cudaStream_t st, bool distinct, bool prefill,
                         bool singles) {
  const ModelSpec& s = spec_;
  const int D = s.d, hd = s.head_dim, nh = s.n_heads, nkv = s.n_kv_heads;
  const float eps = static_cast<float>(s.norm_eps);
  const int* meta = buf_.sel + 2 * max_lrows_;
  // tensor-core path for row buckets >= kTcMinRows (prefill-heavy ticks)
  const bool tc = use_tc_ && tc_ok_ && rcap >= k::kTcMinRows;
  // decode ticks of large models: swap-AB tensor-core GEMV (pure weight stream)
  // (17..64 rows -- incremental-prefill chunks: its wide, N = 32 / 64 variants;
  // MOA_GEMV_MAX_ROWS caps the rows it takes, A/B against the 128-row GEMM tiles)
  static const int gemv_max_rows = [] {
    const char* e = std::getenv("MOA_GEMV_MAX_ROWS");
    return e ? std::max(k::kGemvTcRows, std::min(k::kGemvTcWideRows, std::atoi(e))) : k::kGemvTcWideRows;
  }();
  const bool swap_ab = use_tc_ && tc_ok_ && rcap <= gemv_max_rows;
  const int box = k::gemv_tc_box_rows(rcap);
  auto xmap = [&](const k::TmaMap& m16, const k::TmaMap& m32, const k::TmaMap& m64) {
    return box == k::kGemvTcRows ? &m16 : box == k::kGemvTcMidRows ? &m32 : &m64;
  };
  // decode ticks: RMSNorm folded into the swap-AB GEMV when every normed
  // GEMV of the model qualifies (the residual producers then write ssq)
  const bool norm_fold = swap_ab && nfold_ok_ && use_nfold_;
  auto run_gemm = [&](k::GemvArgs& g, const k::TmaMap* map_a, const k::TmaMap* map_a16, const k::TmaMap& map_w) {
    const bool dec_tc = swap_ab && k::gemv_tc_supported(g);
    if (!tc && !dec_tc) {
      k::gemv(g, st);
      return;
    }
    g.evict_first = evict_first_;
    if (g.X && dec_tc && norm_fold) {  // operand bf16(x) and sums of squares from the residual producer
      g.X = nullptr;
      g.A = hn_;
      g.ssq = ssq_;
      k::gemv_tc(map_w, *xmap(map_hn16_, map_hn32_, map_hn64_), g, gv_ws_, gv_cnt_, st);
      return;
    }
    if (g.X) {  // prep launch: bf16(x) and the rows' inverse RMS, then TMA-load the operand
      k::rmsnorm_rows(g.X, rcap, meta, g.K, inv_, g.eps, hn_, st);
      g.X = nullptr;
      g.A = hn_;
      g.inv = inv_;
      map_a = &map_hn_;
      map_a16 = xmap(map_hn16_, map_hn32_, map_hn64_);
    }
    if (dec_tc)
      k::gemv_tc(map_w, *map_a16, g, gv_ws_, gv_cnt_, st);
    else
      k::gemm_tc(*map_a, map_w, g, st);
  };
  // probes: weight-streaming launches (decode and chunk-tick GEMVs) and prefill-regime ones
  // (tcgen05 GEMM / tiled attention) are separate kinds; bytes are the
  // launch's algorithmic (unique) bytes, flops its dense flops
  auto probe_begin = [&](int kind, double bytes, double flops = 0.0) {
    if (probes_) probes_->begin(kind, bytes, st, flops);
  };
  // (the wide swap-AB GEMVs of 17..64-row chunk ticks stream the weights like
  // decode: HBM-bound kinds; the prefill kinds are the tcgen05 GEMM launches)
  auto gkind = [&](int dec, int pf) { return tc && !swap_ab ? pf : dec; };
  const double Rv = live_R_;
  auto probe_end = [&]() {
    if (probes_) probes_->end(st);
  };
  // decode ticks of small agents: (embedding gather +) RMSNorm + QKV + RoPE + KV
  // append + attention in one launch per layer
  const bool qkv_attn = use_tc_ && use_qkv_attn_ && qkv_attn_ok_ && distinct && rcap <= k::kGemvTcRows;
  const bool fuse_o = qkv_attn && wo_blk_ != nullptr;
  // key splits of the tcgen05 prefill attention (chunk ticks: few row blocks);
  // nsplit bounds the tick's 64-key blocks
  const int pf_ks = pf_tc_ && pf_ws_ ? k::attention_prefill_tc_splits(rcap, nh, nkv, nsplit * split_keys_ / 64) : 1;
  if (!qkv_attn) {  // (the fused QKV + attention kernel gathers layer 0's embeddings itself)
  probe_begin(KernelProbes::Embed, 6.0 * live_R_ * D);
  k::embed(buf_.rows, rcap, meta, out_tok_read, emb_, D, x_, st, norm_fold ? ssq_ : nullptr, norm_fold ? hn_ : nullptr);
  probe_end();
  }
  for (int l = 0; l < s.n_layers; ++l) {
    const Layer& L = layers_[static_cast<std::size_t>(l)];
    const long long loff = layer_stride_ * l;
    if (qkv_attn) {
      // Wqkv (+ Wo when the o-projection is fused), every row's K/V prefix once, x in and out
      probe_begin(KernelProbes::QkvAttn, 2.0 * s.qkv_cols() * D + (fuse_o ? 2.0 * D * nh * hd : 0.0) +
                                             4.0 * live_.keys * nkv * hd + 8.0 * Rv * D);
      k::qkv_attention(x_, ones_, eps, D, L.wqkv, buf_.rows, rcap, meta, rope_, nh, nkv, hd, kpool_, vpool_, kv_stride_,
                       loff, max_ctx_, h_, st, l == 0 ? emb_ : nullptr, out_tok_read, kv_maps_ok_ ? &kmap_ : nullptr,
                       kv_maps_ok_ ? &vmap_ : nullptr, fuse_o ? wo_blk_ + static_cast<long long>(l) * D * nh * hd : nullptr);
      probe_end();
    } else {
    // rmsnorm -> QKV -> RoPE -> KV append
    k::GemvArgs qkv;
    qkv.X = x_;
    qkv.eps = eps;
    qkv.R = rcap;
    qkv.meta = meta;
    qkv.N = s.qkv_cols();
    qkv.K = D;
    qkv.W = L.wqkv;
    qkv.epi = k::kEpiQkv;
    qkv.out_bf16 = q_;
    qkv.rows = buf_.rows;
    qkv.rope = rope_;
    qkv.kpool = kpool_;
    qkv.vpool = vpool_;
    qkv.kv_stride = kv_stride_;
    qkv.layer_off = loff;
    qkv.max_ctx = max_ctx_;
    qkv.nh = nh;
    qkv.nkv = nkv;
    qkv.hd = hd;
    probe_begin(gkind(KernelProbes::Qkv, KernelProbes::PfQkv), 2.0 * qkv.N * qkv.K + 4.0 * Rv * D + 2.0 * Rv * qkv.N,
                2.0 * Rv * qkv.N * qkv.K);
    run_gemm(qkv, nullptr, nullptr, wmaps_[static_cast<std::size_t>(l)].wqkv);
    probe_end();
    // prompt-prefill ticks: runs of a prompt by the tiled kernel (unique bytes:
    // each run's key prefix once; flops: causal QK^T and PV), the tick's decode
    // rows (alone in their run) by the per-row kernel (bytes: each row's prefix)
    if (prefill) {
      const double run_rows = Rv - static_cast<double>(live_.singles);
      probe_begin(KernelProbes::AttnPrefill, 4.0 * live_.run_keys * nkv * hd + 4.0 * run_rows * nh * hd,
                  4.0 * static_cast<double>(live_.run_pairs) * nh * hd);
      if (pf_tc_)
        k::attention_prefill_tc(qmap3_, kmap_, vmap_, buf_.rows, rcap, meta, nh, nkv, hd, kv_stride_, loff, max_ctx_,
                                h_, st, pf_ks, pf_ws_);
      else
        k::attention_prefill(q_, buf_.rows, rcap, meta, nh, nkv, hd, kpool_, vpool_, kv_stride_, loff, max_ctx_, h_,
                             st);
      probe_end();
    }
    if (!prefill || singles) {
      const double keys = prefill ? live_.single_keys : live_.keys, rows_n = prefill ? live_.singles : Rv;
      probe_begin(KernelProbes::AttnDecode, 4.0 * keys * nkv * hd + 4.0 * rows_n * nh * hd,
                  4.0 * keys * nh * hd);
      if (attn_cluster_)
        k::attention_decode_cluster(kmap_, vmap_, q_, buf_.rows, rcap,
                                    k::attention_decode_cluster_splits(rcap, nkv, nsplit), meta, nh, nkv, hd,
                                    kv_stride_, loff, max_ctx_, h_, st, prefill);
      else if (attn_tma_)
        k::attention_decode_tma(kmap_, vmap_, q_, buf_.rows, rcap, nsplit, meta, nh, nkv, hd, kv_stride_, loff,
                                max_ctx_, h_, attn_ws_, attn_cnt_, st, prefill);
      else
        k::attention(q_, buf_.rows, rcap, nsplit, meta, nh, nkv, hd, kpool_, vpool_, kv_stride_, loff, max_ctx_, h_,
                     attn_ws_, attn_cnt_, st, prefill);
      probe_end();
    }
    }
    // x += o . Wo^T (folded into the fused QKV + attention kernel when fuse_o)
    if (!fuse_o) {
    k::GemvArgs o;
    o.A = h_;
    o.R = rcap;
    o.meta = meta;
    o.N = D;
    o.K = nh * hd;
    o.W = L.wo;
    o.epi = k::kEpiResidual;
    o.out = x_;
    // x was last written two kernels back, except when layer 0's fused kernel gathered it
    o.res_early = !(qkv_attn && l == 0);
    if (norm_fold) o.ssq_out = ssq_, o.xb_out = hn_;
    probe_begin(gkind(KernelProbes::OProj, KernelProbes::PfOProj), 2.0 * o.N * o.K + 2.0 * Rv * o.K + 8.0 * Rv * D,
                2.0 * Rv * o.N * o.K);
    run_gemm(o, &map_h_attn_, xmap(map_h_attn16_, map_h_attn32_, map_h_attn64_), wmaps_[static_cast<std::size_t>(l)].wo);
    probe_end();
    }
    // a = silu(gate) * up over rmsnorm(x)
    k::GemvArgs gu;
    gu.X = x_;
    gu.eps = eps;
    gu.R = rcap;
    gu.meta = meta;
    gu.N = 2 * s.ffn;
    gu.K = D;
    gu.W = L.wgu;
    gu.epi = k::kEpiSwiGlu;
    gu.out_bf16 = h_;
    probe_begin(gkind(KernelProbes::GateUp, KernelProbes::PfGateUp), 2.0 * gu.N * gu.K + 4.0 * Rv * D + 2.0 * Rv * s.ffn,
                2.0 * Rv * gu.N * gu.K);
    run_gemm(gu, nullptr, nullptr, wmaps_[static_cast<std::size_t>(l)].wgu);
    probe_end();
    // x += a . Wd^T
    k::GemvArgs dn;
    dn.A = h_;
    dn.R = rcap;
    dn.meta = meta;
    dn.N = D;
    dn.K = s.ffn;
    dn.W = L.wd;
    dn.epi = k::kEpiResidual;
    dn.out = x_;
    dn.res_early = true;  // x was written by the o-projection, two kernels back
    if (norm_fold) dn.ssq_out = ssq_, dn.xb_out = hn_;
    probe_begin(gkind(KernelProbes::Down, KernelProbes::PfDown), 2.0 * dn.N * dn.K + 2.0 * Rv * dn.K + 8.0 * Rv * D,
                2.0 * Rv * dn.N * dn.K);
    run_gemm(dn, &map_h_ffn_, xmap(map_h_ffn16_, map_h_ffn32_, map_h_ffn64_), wmaps_[static_cast<std::size_t>(l)].wd);
    probe_end();
  }
  if (with_logits) {
    probe_begin(KernelProbes::LmHead, 2.0 * s.vocab * D + 4.0 * live_Rl_ * D);
    if (use_tc_ && tc_ok_ && max_lrows_ <= k::kGemvTcRows) {
      // normalise the selected rows, then the swap-AB tensor-core GEMV with
      // the fused greedy-statistics epilogue (LM head = one weight stream)
      k::GemvArgs lm;
      lm.A = hn_;
      static const bool lm_fold = [] {
        const char* e = std::getenv("MOA_LM_FOLD");
        return !(e && e[0] == '0');
      }();
      if (lm_fold) {
        // the LM head normalises its selected rows itself (no rmsnorm launch);
        // on decode ticks from the last residual GEMV's bf16 copy of x and its
        // sums of squares
        lm.X = x_;
        if (norm_fold) lm.ssq = ssq_;
        lm.eps = eps;
        lm.sel = buf_.sel;
      } else {
        k::rmsnorm_rows(x_, max_lrows_, meta, D, inv_, eps, hn_, st, buf_.sel, 1);
        lm.inv = inv_;
      }
      lm.R = k::kGemvTcRows;
      lm.meta = meta + 1;  // live logits rows
      lm.N = s.vocab;
      lm.K = D;
      lm.W = lm_;
      lm.epi = k::kEpiLmStats;
      lm.lm_part = part_;
      lm.lm_cnt = lm_cnt_;
      lm.out_idx = buf_.sel + max_lrows_;
      lm.out_tok = out_tok;
      lm.out_lp = out_lp;
      lm.out_ent = out_ent;
      lm.logits = logits;
      lm.evict_first = evict_first_;
      k::lm_head_tc(wmap_lm_, map_hn16_, lm, part_, lm_cnt_, lm_grid_, st);
    } else {
      k::lm_head(x_, buf_.sel, meta, ones_, eps, lm_, s.vocab, D, part_, lm_cnt_, buf_.sel + max_lrows_, out_tok,
                 out_lp, out_ent, logits, st);
    }
    probe_end();
  }
  MOA_CUDA(cudaGetLastError());
}

void DeviceModel::graphs_clear() {
  for (auto& [key, exec] : graphs_) cudaGraphExecDestroy(exec);
  graphs_.clear();
}

}  // namespace moa
