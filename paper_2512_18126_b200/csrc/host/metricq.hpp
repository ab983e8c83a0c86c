// MetricQ early-exit policy (Algorithm 1).  Host fp64 parts restate
// metricq.cpp:18-131; the per-completion signals (confidence, mock
// embedding, correlation, FCS row) run as device kernels (kernels/ee.cu).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.hpp"

namespace moa {

constexpr double kDefaultTau = 0.7;  // metricq.hpp:15

double geometric_mean_confidence(const std::vector<double>& lp);
double rms_aggregate(const std::vector<double>& c);
// W and P over the lower triangle of an n x n row-major sim matrix.
void weighted_similarity(const std::vector<double>& c, const std::vector<double>& sim, bool diag,
                         double* w, double* p);
double calibrate(double p, double tau);
double quality(double c_bar, double b);

struct QualityScore {
  int outputs = 0;
  std::vector<double> confidences;
  double c_bar = 0, weight_sum = 0, weighted = 0, calibrated = 0, q = 0, tau = kDefaultTau;
  std::vector<double> sim;  // row-major n x n
};

struct ExitDecision {
  double q = 0.0, draw = 1.0;
  bool exited = false;
};
ExitDecision decide_exit(double q, rng::Stream& s);  // metricq.cpp:125-131

// Incremental evaluator for one exit group over device-resident completions
// (metricq.cpp:148-194).  The mock provider (hidden, seed) is the embedding
// source (embedding.cpp:86-120), or the caller writes the rows into
// emb_buffer() (hidden-state / external providers).  Groups whose width
// exceeds their longest completion (h > n) use the n x n cross-Gram route
// (kernels/ee.cu): per completion the column-normalised rows and the norm of
// its correlation are kept instead of an h x h correlation matrix.
class GpuMetricQ {
 public:
  GpuMetricQ(int hidden, std::uint64_t seed, double tau, bool include_diagonal, int max_members,
             int max_tokens, cudaStream_t st);
  ~GpuMetricQ();
  GpuMetricQ(const GpuMetricQ&) = delete;
  GpuMetricQ& operator=(const GpuMetricQ&) = delete;

  // Completion = n device tokens at d_tok[base..] with fp32 logprobs at
  // d_lp[base..].  Synchronises the stream once (reads C and the sim row).
  QualityScore add_completion(const int* d_tok, const float* d_lp, long long base, int n);
  // Same with the embedding rows already in emb_buffer() (hidden-state provider).
  QualityScore add_completion_embedded(const float* d_lp, long long base, int n);
  // Same with host embedding rows emb[n][hidden] (a caller EmbeddingProvider).
  QualityScore add_completion_host(const double* emb, const float* d_lp, long long base, int n);
  // Embedding rows already in emb_buffer(), confidence computed by the caller
  // (host fp64 logprobs: geometric_mean_confidence, bit-exact).
  QualityScore add_completion_conf(double c, int n);
  bool cross_route() const { return cross_; }
  double* emb_buffer() { return d_emb_; }
  int hidden() const { return hidden_; }
  int completions() const { return static_cast<int>(conf_.size()); }
  // Reuse the device buffers for a new group (no reallocation).
  bool fits(int hidden, int max_members, int max_tokens) const {
    return hidden == hidden_ && max_members <= max_members_ && max_tokens <= max_tokens_;
  }
  void reset(std::uint64_t seed, double tau, bool include_diagonal) {
    seed_ = seed;
    tau_ = tau;
    diag_ = include_diagonal;
    conf_.clear();
    sim_.clear();
    nv_.clear();
    self_.clear();
  }

 private:
  QualityScore finish(const float* d_lp, long long base, int n, const double* conf = nullptr, bool computed = false);
  QualityScore current() const;
  int hidden_;
  std::uint64_t seed_;
  double tau_;
  bool diag_;
  int max_members_, max_tokens_;
  cudaStream_t st_;
  double* d_emb_ = nullptr;    // [max_tokens][h]
  double* d_gram_ = nullptr;   // [h][h]
  double* d_corrs_ = nullptr;  // [max_members][h][h]
  double* d_out_ = nullptr;    // [1 + max_members]: C, sim row
  double* h_out_ = nullptr;    // pinned mirror
  std::vector<double> conf_;
  std::vector<double> sim_;  // n x n
  // n x n route (hidden_ > max_tokens_)
  bool cross_ = false;
  bool fused_ = true;  // mock provider, h x h route: one launch per evaluation (ee_fused_mock)
  double* d_hat_ = nullptr;   // [max_members][max_tokens][h] column-normalised rows
  int* d_nv_ = nullptr;       // [max_members] rows per stored completion
  double* d_part_ = nullptr;  // per-tile partial sums of squares
  std::vector<int> nv_;
  std::vector<double> self_;  // ||Corr||_F per stored completion
};

}  // namespace moa
