#include "metricq.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "../kernels/kernels.cuh"
#include "model.hpp"

namespace moa {

double geometric_mean_confidence(const std::vector<double>& lp) {
  if (lp.empty()) throw ValidationError("logprobs: need at least one token");
  double s = 0.0;
  for (double v : lp) {
    if (!std::isfinite(v)) throw ValidationError("logprobs: values must be finite");
    if (v > 0.0) throw ValidationError("logprobs: values must be <= 0");
    s += v;
  }
  return std::exp(s / static_cast<double>(lp.size()));
}

double rms_aggregate(const std::vector<double>& c) {
  if (c.empty()) throw ValidationError("rms_aggregate: empty confidence set");
  double s = 0.0;
  for (double v : c) s += v * v;
  return std::sqrt(s / static_cast<double>(c.size()));
}

void weighted_similarity(const std::vector<double>& c, const std::vector<double>& sim, bool diag,
                         double* w, double* p) {
  const std::size_t n = c.size();
  if (sim.size() != n * n) throw ValidationError("weighted_similarity: sim matrix does not match confidence count");
  double ws = 0.0, acc = 0.0;
  for (std::size_t i = 0; i < n; ++i) {
    const std::size_t jend = diag ? i + 1 : i;
    for (std::size_t j = 0; j < jend; ++j) {
      const double wij = c[i] * c[j];
      ws += wij;
      acc += wij * sim[i * n + j];
    }
  }
  *w = ws;
  *p = ws > 0.0 ? acc / ws : 0.0;
}

double calibrate(double p, double tau) {
  if (!(tau > 0.0)) throw ValidationError("calibrate: tau must be > 0");
  return std::clamp(1.0 - std::abs(p - tau) / tau, 0.0, 1.0);
}

double quality(double c_bar, double b) { return std::sqrt(c_bar * b); }

ExitDecision decide_exit(double q, rng::Stream& s) {
  ExitDecision d;
  d.q = q;
  d.draw = s.next_uniform();
  d.exited = d.draw < q;
  return d;
}

GpuMetricQ::GpuMetricQ(int hidden, std::uint64_t seed, double tau, bool include_diagonal, int max_members,
                       int max_tokens, cudaStream_t st)
    : hidden_(hidden), seed_(seed), tau_(tau), diag_(include_diagonal), max_members_(max_members),
      max_tokens_(max_tokens), st_(st) {
  if (!(tau > 0.0 && tau <= 1.0)) throw ValidationError("metricq: tau must be in (0, 1]");
  if (hidden <= 0) throw ValidationError("provider.hidden: must be > 0");
  const long long hh = static_cast<long long>(hidden) * hidden;
  MOA_CUDA(cudaMalloc(&d_emb_, sizeof(double) * static_cast<long long>(max_tokens) * hidden));
  cross_ = hidden > max_tokens;
  if (const char* e = std::getenv("MOA_FCS_ROUTE")) cross_ = std::string(e) == "nn";  // force one route (tests)
  if (const char* e = std::getenv("MOA_EE_FUSED")) fused_ = std::string(e) != "0";    // A/B: the 5-launch path
  if (cross_) {
    MOA_CUDA(cudaMalloc(&d_hat_, sizeof(double) * static_cast<long long>(max_members) * max_tokens * hidden));
    MOA_CUDA(cudaMalloc(&d_nv_, sizeof(int) * max_members));
    MOA_CUDA(cudaMalloc(&d_part_, sizeof(double) * k::ee_cross_parts(max_tokens, max_members)));
  } else {
    MOA_CUDA(cudaMalloc(&d_gram_, sizeof(double) * hh));
    MOA_CUDA(cudaMalloc(&d_corrs_, sizeof(double) * hh * max_members));
  }
  MOA_CUDA(cudaMalloc(&d_out_, sizeof(double) * (1 + max_members)));
  MOA_CUDA(cudaMallocHost(&h_out_, sizeof(double) * (1 + max_members)));
}

GpuMetricQ::~GpuMetricQ() {
  for (void* p : {static_cast<void*>(d_emb_), static_cast<void*>(d_gram_), static_cast<void*>(d_corrs_),
                  static_cast<void*>(d_out_), static_cast<void*>(d_hat_), static_cast<void*>(d_nv_),
                  static_cast<void*>(d_part_)})
    if (p) cudaFree(p);
  if (h_out_) cudaFreeHost(h_out_);
}

QualityScore GpuMetricQ::add_completion(const int* d_tok, const float* d_lp, long long base, int n) {
  if (n <= 0) throw ValidationError("logprobs: need at least one token");
  if (n > max_tokens_) throw ValidationError("metricq: completion longer than the evaluator capacity");
  if (!cross_ && fused_ && k::ee_fused_mock_supported(hidden_, completions())) {
    // the whole evaluation in one launch; one synchronisation for its result
    const int m = completions();
    if (m >= max_members_) throw ValidationError("metricq: exit group capacity exceeded");
    k::ee_fused_mock(d_tok, d_lp, base, n, hidden_, seed_, 1e-12, d_corrs_, m, d_out_, st_);
    return finish(nullptr, 0, n, nullptr, true);
  }
  k::ee_mock_embed(d_tok, base, n, hidden_, seed_, d_emb_, st_);
  return finish(d_lp, base, n);
}

QualityScore GpuMetricQ::add_completion_embedded(const float* d_lp, long long base, int n) {
  if (n <= 0) throw ValidationError("logprobs: need at least one token");
  if (n > max_tokens_) throw ValidationError("metricq: completion longer than the evaluator capacity");
  return finish(d_lp, base, n);
}

QualityScore GpuMetricQ::add_completion_host(const double* emb, const float* d_lp, long long base, int n) {
  if (n <= 0) throw ValidationError("logprobs: need at least one token");
  if (n > max_tokens_) throw ValidationError("metricq: completion longer than the evaluator capacity");
  MOA_CUDA(cudaMemcpyAsync(d_emb_, emb, sizeof(double) * n * hidden_, cudaMemcpyHostToDevice, st_));
  return finish(d_lp, base, n);
}

QualityScore GpuMetricQ::add_completion_conf(double c, int n) {
  if (n <= 0) throw ValidationError("logprobs: need at least one token");
  if (n > max_tokens_) throw ValidationError("metricq: completion longer than the evaluator capacity");
  return finish(nullptr, 0, n, &c);
}

QualityScore GpuMetricQ::finish(const float* d_lp, long long base, int n, const double* conf, bool computed) {
  const int m = completions();
  if (m >= max_members_) throw ValidationError("metricq: exit group capacity exceeded");
  const long long hh = static_cast<long long>(hidden_) * hidden_;
  if (!conf && !computed) k::ee_confidence(d_lp + base, n, d_out_, st_);
  const int nout = cross_ ? 2 + m : 1 + m;  // C, FCS numerators (+ the self term on the n x n route)
  if (computed) {
    // d_out_ already holds C and the FCS row (ee_fused_mock)
  } else if (cross_) {
    const long long stride = static_cast<long long>(max_tokens_) * hidden_;
    double* hat = d_hat_ + stride * m;
    k::ee_colnorm(d_emb_, n, hidden_, 1e-12, hat, st_);
    MOA_CUDA(cudaMemcpyAsync(d_nv_ + m, &n, sizeof(int), cudaMemcpyHostToDevice, st_));
    const int nmax = nv_.empty() ? n : std::max(n, *std::max_element(nv_.begin(), nv_.end()));
    k::ee_cross_sumsq(hat, n, d_hat_, d_nv_, nmax, stride, m, hidden_, d_part_, d_out_ + 1, st_);
  } else {
    double* corr_new = d_corrs_ + hh * m;
    k::ee_corr(d_emb_, n, hidden_, 1e-12, d_gram_, corr_new, st_);
    k::ee_fcs(corr_new, d_corrs_, m, hidden_, d_out_ + 1, st_);
  }
  MOA_CUDA(cudaMemcpyAsync(h_out_, d_out_, sizeof(double) * nout, cudaMemcpyDeviceToHost, st_));
  MOA_CUDA(cudaStreamSynchronize(st_));
  MOA_CUDA(cudaGetLastError());
  const double c = conf ? *conf : h_out_[0];
  if (cross_) {  // frob_cos_sim_corr from the cross / self sums of squares (metricq.cpp:55-64)
    const double self = std::sqrt(h_out_[1 + m]);
    for (int j = 0; j < m; ++j)
      h_out_[1 + j] = (self == 0.0 || self_[static_cast<std::size_t>(j)] == 0.0)
                          ? 0.0
                          : h_out_[1 + j] / (self * self_[static_cast<std::size_t>(j)]);
    self_.push_back(self);
    nv_.push_back(n);
  }
  if (!std::isfinite(c) || c > 1.0) throw ValidationError("logprobs: values must be finite and <= 0");
  // grow the sim matrix by one row/column (metricq.cpp:159-168)
  const int nn = m + 1;
  std::vector<double> grown(static_cast<std::size_t>(nn) * nn, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) grown[static_cast<std::size_t>(i) * nn + j] = sim_[static_cast<std::size_t>(i) * m + j];
  grown[static_cast<std::size_t>(m) * nn + m] = 1.0;
  for (int j = 0; j < m; ++j) {
    grown[static_cast<std::size_t>(m) * nn + j] = h_out_[1 + j];
    grown[static_cast<std::size_t>(j) * nn + m] = h_out_[1 + j];
  }
  sim_.swap(grown);
  conf_.push_back(c);
  return current();
}

QualityScore GpuMetricQ::current() const {
  QualityScore qs;
  qs.outputs = completions();
  qs.confidences = conf_;
  qs.c_bar = rms_aggregate(conf_);
  qs.sim = sim_;
  weighted_similarity(conf_, sim_, diag_, &qs.weight_sum, &qs.weighted);
  qs.calibrated = calibrate(qs.weighted, tau_);
  qs.q = quality(qs.c_bar, qs.calibrated);
  qs.tau = tau_;
  return qs;
}

}  // namespace moa
