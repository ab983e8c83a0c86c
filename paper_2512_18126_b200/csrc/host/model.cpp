#include "model.hpp"

#include <algorithm>
#include <cmath>

namespace moa {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

long long ModelSpec::weight_elems() const {
  const long long D = d, hd = head_dim;
  long long per_layer = qkv_cols() * D + D * n_heads * hd + 2LL * ffn * D + D * ffn;
  return 2LL * vocab * D + n_layers * per_layer;
}

void ModelSpec::validate() const {
  if (d <= 0 || n_layers <= 0 || n_heads <= 0 || n_kv_heads <= 0 || ffn <= 0 || vocab <= 0)
    throw ValidationError("model " + tag + ": dimensions must be positive");
  if (head_dim != 64 && head_dim != 128) throw ValidationError("model " + tag + ": head_dim must be 64 or 128");
  if (n_heads % n_kv_heads) throw ValidationError("model " + tag + ": n_heads % n_kv_heads != 0");
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

}  // namespace

DeviceModel::DeviceModel(const ModelSpec& spec, int max_agents, int max_ctx, int max_rows,
                         int max_logit_rows, cudaStream_t st)
    : spec_(spec), max_agents_(max_agents), max_ctx_(max_ctx), max_rows_(max_rows),
      max_lrows_(max_logit_rows) {
  spec_.validate();
  const ModelSpec& s = spec_;
  const long long D = s.d, hd = s.head_dim, V = s.vocab;
  MOA_CUDA(cudaMalloc(&wbase_, sizeof(k::bf16) * s.weight_elems()));
  k::bf16* p = wbase_;
  auto take = [&](long long n) {
    k::bf16* r = p;
    p += n;
    return r;
  };
  auto init = [&](k::bf16* dst, const std::string& name, long long rows, long long cols) {
    k::init_uniform(dst, rows * cols, tensor_base(s, name), tensor_scale(s, name, static_cast<int>(cols)), st);
  };
  emb_ = take(V * D);
  init(emb_, "emb", V, D);
  for (int l = 0; l < s.n_layers; ++l) {
    Layer L{};
    const std::string pre = "L" + std::to_string(l) + ".";
    L.wqkv = take(s.qkv_cols() * D);
    init(L.wqkv, pre + "wq", s.n_heads * hd, D);
    init(L.wqkv + s.n_heads * hd * D, pre + "wk", s.n_kv_heads * hd, D);
    init(L.wqkv + (s.n_heads + s.n_kv_heads) * hd * D, pre + "wv", s.n_kv_heads * hd, D);
    L.wo = take(D * s.n_heads * hd);
    init(L.wo, pre + "wo", D, s.n_heads * hd);
    L.wgu = take(2LL * s.ffn * D);
    init(L.wgu, pre + "wg", s.ffn, D);
    init(L.wgu + static_cast<long long>(s.ffn) * D, pre + "wu", s.ffn, D);
    L.wd = take(D * s.ffn);
    init(L.wd, pre + "wd", D, s.ffn);
    layers_.push_back(L);
  }
  lm_ = take(V * D);
  init(lm_, "lm", V, D);

  const int maxd = std::max({s.d, s.ffn, s.n_heads * s.head_dim});
  MOA_CUDA(cudaMalloc(&ones_, sizeof(float) * maxd));
  k::fill_f32(ones_, maxd, 1.0f, st);

  // RoPE table in fp64 libm then one cast (identical to oracle/model.py rope_table)
  const int half = s.head_dim / 2;
  std::vector<float2> tab(static_cast<std::size_t>(max_ctx) * half);
  for (int pos = 0; pos < max_ctx; ++pos)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(s.rope_theta, -2.0 * i / s.head_dim);
      const double a = pos * inv;
      tab[static_cast<std::size_t>(pos) * half + i] = make_float2(static_cast<float>(std::cos(a)),
                                                                  static_cast<float>(std::sin(a)));
    }
  MOA_CUDA(cudaMalloc(&rope_, sizeof(float2) * tab.size()));
  MOA_CUDA(cudaMemcpyAsync(rope_, tab.data(), sizeof(float2) * tab.size(), cudaMemcpyHostToDevice, st));

  layer_stride_ = static_cast<long long>(s.n_kv_heads) * max_ctx * hd;
  kv_stride_ = layer_stride_ * s.n_layers;
  MOA_CUDA(cudaMalloc(&kpool_, sizeof(k::bf16) * kv_stride_ * max_agents));
  MOA_CUDA(cudaMalloc(&vpool_, sizeof(k::bf16) * kv_stride_ * max_agents));

  MOA_CUDA(cudaMalloc(&x_, sizeof(float) * static_cast<long long>(max_rows) * D));
  MOA_CUDA(cudaMalloc(&h_, sizeof(k::bf16) * static_cast<long long>(max_rows) * maxd));
  MOA_CUDA(cudaMalloc(&q_, sizeof(k::bf16) * static_cast<long long>(max_rows) * s.n_heads * hd));
  const long long ncap = std::max({static_cast<long long>(s.qkv_cols()), 2LL * s.ffn, D});
  P_cap_ = std::max(max_rows, 128) * ncap;
  MOA_CUDA(cudaMalloc(&P_, sizeof(float) * P_cap_));
  MOA_CUDA(cudaMalloc(&part_, sizeof(k::LmStat) * static_cast<long long>(max_logit_rows) * k::lm_head_blocks(s.vocab)));
  MOA_CUDA(cudaMalloc(&buf_.rows, sizeof(k::RowDesc) * max_rows));
  MOA_CUDA(cudaMalloc(&buf_.sel, sizeof(int) * 2 * max_logit_rows));
  MOA_CUDA(cudaGetLastError());
}

DeviceModel::~DeviceModel() {
  for (void* ptr : {static_cast<void*>(wbase_), static_cast<void*>(ones_), static_cast<void*>(rope_),
                    static_cast<void*>(kpool_), static_cast<void*>(vpool_), static_cast<void*>(x_),
                    static_cast<void*>(h_), static_cast<void*>(q_), static_cast<void*>(P_),
                    static_cast<void*>(part_), static_cast<void*>(buf_.rows),
                    static_cast<void*>(buf_.sel)})
    if (ptr) cudaFree(ptr);
}

int DeviceModel::bind_agent() {
  if (bound_ >= max_agents_)
    throw ValidationError("model " + spec_.tag + ": agent capacity " + std::to_string(max_agents_) +
                          " exhausted");
  return bound_++;
}

// Split K until one row block's grid covers ~2 waves of 148 SMs.  S depends
// on (N, K) only, never on the batch, so a row's result is bit-identical
// whichever rows share its tick (batch invariance: schedule modes decode the
// same tokens).  The consumer kernel sums the S partial slices in order.
int DeviceModel::split_k(int N, int K, int R) const {
  const long long blocks = (N + 31) / 32;
  int S = 1;
  while (blocks * S < 296 && (K / (S * 2)) % 256 == 0 && K / (S * 2) >= 256 && S < 16) S *= 2;
  while (S > 1 && static_cast<long long>(S) * R * N > P_cap_) S /= 2;
  return S;
}

void DeviceModel::forward(int R, int Rl, const int* out_tok_read, int* out_tok, float* out_lp,
                          float* out_ent, float* logits, cudaStream_t st) {
  if (R <= 0) return;
  if (R > max_rows_) throw RunError("model " + spec_.tag + ": tick rows exceed workspace");
  const ModelSpec& s = spec_;
  const int D = s.d, hd = s.head_dim, nh = s.n_heads, nkv = s.n_kv_heads;
  const float eps = static_cast<float>(s.norm_eps);
  k::embed(buf_.rows, R, out_tok_read, emb_, D, x_, st);
  for (int l = 0; l < s.n_layers; ++l) {
    const Layer& L = layers_[static_cast<std::size_t>(l)];
    const long long loff = layer_stride_ * l;
    k::rmsnorm(x_, nullptr, R, D, ones_, eps, h_, st);
    int S = split_k(s.qkv_cols(), D, R);
    k::gemm_skinny(h_, R, L.wqkv, s.qkv_cols(), D, S, P_, st);
    k::rope_kv(P_, S, buf_.rows, R, nh, nkv, hd, rope_, q_, kpool_, vpool_, kv_stride_, loff, max_ctx_, st);
    k::attention(q_, buf_.rows, R, nh, nkv, hd, kpool_, vpool_, kv_stride_, loff, max_ctx_, h_, st);
    S = split_k(D, nh * hd, R);
    k::gemm_skinny(h_, R, L.wo, D, nh * hd, S, P_, st);
    k::residual_add(x_, P_, S, R, D, st);
    k::rmsnorm(x_, nullptr, R, D, ones_, eps, h_, st);
    S = split_k(2 * s.ffn, D, R);
    k::gemm_skinny(h_, R, L.wgu, 2 * s.ffn, D, S, P_, st);
    k::swiglu(P_, S, R, s.ffn, h_, st);
    S = split_k(D, s.ffn, R);
    k::gemm_skinny(h_, R, L.wd, D, s.ffn, S, P_, st);
    k::residual_add(x_, P_, S, R, D, st);
  }
  if (Rl > 0) {
    if (Rl > max_lrows_) throw RunError("model " + spec_.tag + ": logits rows exceed workspace");
    k::rmsnorm(x_, buf_.sel, Rl, D, ones_, eps, h_, st);
    k::lm_head_stats(h_, Rl, lm_, s.vocab, D, part_, logits, st);
    k::lm_merge(part_, Rl, k::lm_head_blocks(s.vocab), buf_.sel + max_lrows_, out_tok, out_lp, out_ent, st);
  }
  MOA_CUDA(cudaGetLastError());
}

}  // namespace moa
