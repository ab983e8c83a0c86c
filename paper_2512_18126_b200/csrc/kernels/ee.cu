// Early-exit signal kernels (fp64 on B200's FP64 pipe):
//   confidence  C = exp(mean logprob)            metricq.cpp:18-23
//   mock embed  hash rows, row-centred           embedding.cpp:91-113 (bit-exact)
//   corr        cosine-normalised Gram t^T t     metricq.cpp:32-53, :157
//   FCS         Frobenius cosine of two corrs    metricq.cpp:55-64
// Two formulations of the FCS (SURVEY.md §7 "FCS at model width"):
//   h x h (h <= n, e.g. the preset mock h = 64): the reference's own route,
//     Gram t^T t -> correlation -> Frobenius cosine of two h x h matrices;
//   n x n (h > n, hidden-state widths): A_hat = A D^-1/2 (dead columns zero),
//     <Corr U, Corr V>_F = ||A_hat B_hat^T||_F^2 and ||Corr U||_F =
//     ||A_hat A_hat^T||_F -- n_u x n_v dot products of length h instead of
//     two h x h matrices per completion.
#include "kernels.cuh"

namespace moa::k {

namespace {

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {
  return mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

__global__ void confidence_kernel(const float* __restrict__ lp, int n, double* __restrict__ c) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += static_cast<double>(lp[i]);  // sequential, as the reference
    *c = exp(s / static_cast<double>(n));
  }
}

__global__ void mock_embed_kernel(const int* __restrict__ out_tok, long long base, int h,
                                  std::uint64_t seed, double* __restrict__ emb) {
  extern __shared__ double row[];
  const int r = blockIdx.x;
  const std::uint64_t tok = static_cast<std::uint64_t>(static_cast<std::int64_t>(out_tok[base + r]));
  const std::uint64_t row_seed = hash_combine(hash_combine(seed, tok), static_cast<std::uint64_t>(r));
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    const std::uint64_t bits = mix64(hash_combine(row_seed, static_cast<std::uint64_t>(c)));
    const double u = static_cast<double>(bits >> 11) * 0x1.0p-53;
    row[c] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
  }
  __syncthreads();
  __shared__ double mean;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int c = 0; c < h; ++c) s += row[c];  // sequential row mean (embedding.cpp:104-108)
    mean = s / static_cast<double>(h);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < h; c += blockDim.x)
    emb[static_cast<long long>(r) * h + c] = row[c] - mean;
}

// gram[i][j] = sum_r emb[r][i] * emb[r][j], sequential in r; mirrored so the
// matrix is exactly symmetric.
__global__ void gram_kernel(const double* __restrict__ emb, int n, int h, double* __restrict__ gram) {
  const long long total = static_cast<long long>(h) * h;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(t / h), j = static_cast<int>(t % h);
    if (j < i) continue;
    double s = 0.0;
    for (int r = 0; r < n; ++r) s = __dadd_rn(s, __dmul_rn(emb[r * h + i], emb[r * h + j]));
    gram[static_cast<long long>(i) * h + j] = s;
    gram[static_cast<long long>(j) * h + i] = s;
  }
}

__global__ void corr_kernel(const double* __restrict__ gram, int h, double eps, double* __restrict__ corr) {
  const long long total = static_cast<long long>(h) * h;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = static_cast<int>(t / h), j = static_cast<int>(t % h);
    const double gi = gram[static_cast<long long>(i) * h + i], gj = gram[static_cast<long long>(j) * h + j];
    double v = 0.0;
    if (gi > eps && gj > eps) {
      if (i == j) {
        v = 1.0;
      } else {
        const int a = i < j ? i : j, b = i < j ? j : i;  // reference computes the upper triangle
        v = gram[static_cast<long long>(a) * h + b] / sqrt(gram[static_cast<long long>(a) * h + a] *
                                                           gram[static_cast<long long>(b) * h + b]);
      }
    }
    corr[t] = v;
  }
}

__global__ void fcs_kernel(const double* __restrict__ cu, const double* __restrict__ corrs, int h,
                           double* __restrict__ sim) {
  __shared__ double red[3][32];
  const int j = blockIdx.x;
  const double* cv = corrs + static_cast<long long>(j) * h * h;
  double dot = 0.0, nu = 0.0, nv = 0.0;
  const long long total = static_cast<long long>(h) * h;
  for (long long t = threadIdx.x; t < total; t += blockDim.x) {
    const double a = cu[t], b = cv[t];
    dot = fma(a, b, dot);
    nu = fma(a, a, nu);
    nv = fma(b, b, nv);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, o);
    nu += __shfl_xor_sync(0xffffffffu, nu, o);
    nv += __shfl_xor_sync(0xffffffffu, nv, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = dot;
    red[1][w] = nu;
    red[2][w] = nv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double d = 0, a = 0, b = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) {
      d += red[0][i];
      a += red[1][i];
      b += red[2][i];
    }
    const double su = sqrt(a), sv = sqrt(b);
    sim[j] = (su == 0.0 || sv == 0.0) ? 0.0 : d / (su * sv);
  }
}

// A_hat[r][c] = A[r][c] / sqrt(sum_r A[r][c]^2), 0 for columns <= eps (the
// reference's dead-column rule, metricq.cpp:32-53); column sums sequential in r.
__global__ void colnorm_kernel(const double* __restrict__ a, int n, int h, double eps, double* __restrict__ ahat) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
  double g = 0.0;
  for (int r = 0; r < n; ++r) {
    const double v = a[static_cast<long long>(r) * h + c];
    g = __dadd_rn(g, __dmul_rn(v, v));
  }
  const double inv = g > eps ? 1.0 / sqrt(g) : 0.0;
  for (int r = 0; r < n; ++r) ahat[static_cast<long long>(r) * h + c] = a[static_cast<long long>(r) * h + c] * inv;
}

// Sum of squares of X = U V_j^T (U: nu x h, V_j: the j-th stored completion,
// nv[j] x h) per 32 x 32 output tile -> part[j][tile] (fixed order in-CTA);
// blockIdx.z = j (j == m: V = U itself, the self term).
constexpr int kXT = 32;
__global__ void __launch_bounds__(256) cross_sumsq_kernel(const double* __restrict__ u, int nu,
                                                          const double* __restrict__ vs, const int* __restrict__ nv,
                                                          long long vstride, int m, int h, double* __restrict__ part,
                                                          int tiles) {
  __shared__ double As[kXT][kXT + 1], Bs[kXT][kXT + 1];
  __shared__ double red[8];
  const int j = blockIdx.z;
  const double* v = j == m ? u : vs + vstride * j;
  const int n2 = j == m ? nu : nv[j];
  const int a0 = blockIdx.x * kXT, b0 = blockIdx.y * kXT;
  const int tile = blockIdx.y * gridDim.x + blockIdx.x;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // output (a0 + ty + 8i, b0 + tx)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (a0 < nu && b0 < n2) {
    for (int k0 = 0; k0 < h; k0 += kXT) {
      for (int e = threadIdx.x; e < kXT * kXT; e += 256) {
        const int rr = e / kXT, kk = e % kXT;
        As[rr][kk] = (a0 + rr < nu && k0 + kk < h) ? u[static_cast<long long>(a0 + rr) * h + k0 + kk] : 0.0;
        Bs[rr][kk] = (b0 + rr < n2 && k0 + kk < h) ? v[static_cast<long long>(b0 + rr) * h + k0 + kk] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int kk = 0; kk < kXT; ++kk) {
        const double b = Bs[tx][kk];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = fma(As[ty + 8 * i][kk], b, acc[i]);
      }
      __syncthreads();
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s = fma(acc[i], acc[i], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (tx == 0) red[ty] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[static_cast<long long>(j) * tiles + tile] = t;
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int tiles, double* __restrict__ out) {
  const int j = blockIdx.x;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < tiles; ++i) t += part[static_cast<long long>(j) * tiles + i];
    out[j] = t;
  }
}

// One launch for a whole mock-provider evaluation on the h x h route (h <=
// 128, <= 16 stored members): confidence (warp 31, sequential fp64 sum), the
// MockProvider rows hashed 32 at a time into shared memory (bit-exact with
// mock_embed_kernel), the Gram's upper triangle accumulated in registers
// (each entry sequential in r, as gram_kernel), the correlation (written to
// corrs[m]) and its Frobenius cosine against every stored member (fixed
// thread -> entry map and reduction tree: deterministic).  out[0] = C,
// out[1 + k] = FCS(new, member k).
constexpr int kEeThreads = 1024, kEeWorkers = 992, kEeRows = 32, kEeMaxM = 16, kEeMaxH = 128;
constexpr int kEeMaxE = kEeMaxH * (kEeMaxH + 1) / 2;
constexpr int kEePer = (kEeMaxE + kEeWorkers - 1) / kEeWorkers;  // entries per worker thread

__global__ void __launch_bounds__(kEeThreads, 1)
ee_fused_mock_kernel(const int* __restrict__ out_tok, const float* __restrict__ lp, long long base, int n, int h,
                     std::uint64_t seed, double eps, double* __restrict__ corrs, int m, double* __restrict__ out) {
  extern __shared__ double ee_sm[];
  double* rows = ee_sm;                                // [kEeRows][h]
  double* diag = rows + kEeRows * h;                   // [h]
  double* mean = diag + h;                             // [kEeRows]
  std::uint32_t* pairs = reinterpret_cast<std::uint32_t*>(mean + kEeRows);  // [E]: i << 16 | j
  __shared__ double red[kEeWorkers / 32][2 * kEeMaxM + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int E = h * (h + 1) / 2;
  const long long hh = static_cast<long long>(h) * h;
  if (warp == kEeWorkers / 32) {  // confidence C = exp(mean logprob), sequential as the reference
    if (lane == 0) {
      double sacc = 0.0;
      for (int i = 0; i < n; ++i) sacc += static_cast<double>(lp[base + i]);
      out[0] = exp(sacc / static_cast<double>(n));
    }
    return;
  }
  for (int e = tid; e < E; e += kEeWorkers) {  // upper-triangle entry table
    int i = 0, rem = e;
    while (rem >= h - i) {
      rem -= h - i;
      ++i;
    }
    pairs[e] = (static_cast<std::uint32_t>(i) << 16) | static_cast<std::uint32_t>(i + rem);
  }
  double acc[kEePer];
#pragma unroll
  for (int k = 0; k < kEePer; ++k) acc[k] = 0.0;
  asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
  for (int r0 = 0; r0 < n; r0 += kEeRows) {
    const int rc = min(kEeRows, n - r0);
    for (int idx = tid; idx < rc * h; idx += kEeWorkers) {
      const int r = idx / h, c = idx % h;
      const std::uint64_t tok = static_cast<std::uint64_t>(static_cast<std::int64_t>(out_tok[base + r0 + r]));
      const std::uint64_t row_seed = hash_combine(hash_combine(seed, tok), static_cast<std::uint64_t>(r0 + r));
      const std::uint64_t bits = mix64(hash_combine(row_seed, static_cast<std::uint64_t>(c)));
      const double u = static_cast<double>(bits >> 11) * 0x1.0p-53;
      rows[r * h + c] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
    if (tid < rc) {  // sequential row mean (embedding.cpp:104-108)
      double sm = 0.0;
      for (int c = 0; c < h; ++c) sm += rows[tid * h + c];
      mean[tid] = sm / static_cast<double>(h);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
    for (int idx = tid; idx < rc * h; idx += kEeWorkers) rows[idx] = rows[idx] - mean[idx / h];
    asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
#pragma unroll
    for (int k = 0; k < kEePer; ++k) {
      const int e = tid + k * kEeWorkers;
      if (e >= E) break;
      const int i = pairs[e] >> 16, j = pairs[e] & 0xffff;
      double a = acc[k];
      for (int r = 0; r < rc; ++r) a = __dadd_rn(a, __dmul_rn(rows[r * h + i], rows[r * h + j]));
      acc[k] = a;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
  }
#pragma unroll
  for (int k = 0; k < kEePer; ++k) {
    const int e = tid + k * kEeWorkers;
    if (e < E && (pairs[e] >> 16) == (pairs[e] & 0xffff)) diag[pairs[e] >> 16] = acc[k];
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
  // correlation (metricq.cpp:32-53, upper triangle mirrored) and the FCS sums
  double dot[kEeMaxM], nv[kEeMaxM], nu = 0.0;
#pragma unroll
  for (int k = 0; k < kEeMaxM; ++k) dot[k] = nv[k] = 0.0;
  double* cnew = corrs + hh * m;
#pragma unroll
  for (int k = 0; k < kEePer; ++k) {
    const int e = tid + k * kEeWorkers;
    if (e >= E) break;
    const int i = pairs[e] >> 16, j = pairs[e] & 0xffff;
    const double gi = diag[i], gj = diag[j];
    double v = 0.0;
    if (gi > eps && gj > eps) v = i == j ? 1.0 : acc[k] / sqrt(gi * gj);
    cnew[static_cast<long long>(i) * h + j] = v;
    cnew[static_cast<long long>(j) * h + i] = v;
    const double w = i == j ? 1.0 : 2.0;  // symmetric: off-diagonal entries count twice
    nu = fma(w * v, v, nu);
#pragma unroll
    for (int q = 0; q < kEeMaxM; ++q) {
      if (q >= m) break;
      const double b = corrs[hh * q + static_cast<long long>(i) * h + j];
      dot[q] = fma(w * v, b, dot[q]);
      nv[q] = fma(w * b, b, nv[q]);
    }
  }
  // reduction: warp shuffles, then warps in order
#pragma unroll
  for (int o = 16; o; o >>= 1) nu += __shfl_xor_sync(0xffffffffu, nu, o);
#pragma unroll
  for (int q = 0; q < kEeMaxM; ++q) {
    if (q >= m) break;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      dot[q] += __shfl_xor_sync(0xffffffffu, dot[q], o);
      nv[q] += __shfl_xor_sync(0xffffffffu, nv[q], o);
    }
  }
  if (lane == 0) {
    red[warp][2 * kEeMaxM] = nu;
    for (int q = 0; q < m; ++q) {
      red[warp][q] = dot[q];
      red[warp][kEeMaxM + q] = nv[q];
    }
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kEeWorkers) : "memory");
  if (tid < m) {
    double d = 0.0, a = 0.0, b = 0.0;
    for (int w = 0; w < kEeWorkers / 32; ++w) {
      d += red[w][tid];
      a += red[w][2 * kEeMaxM];
      b += red[w][kEeMaxM + tid];
    }
    const double su = sqrt(a), sv = sqrt(b);
    out[1 + tid] = (su == 0.0 || sv == 0.0) ? 0.0 : d / (su * sv);
  }
}

}  // namespace

void ee_colnorm(const double* emb, int n, int h, double eps, double* ahat, cudaStream_t st) {
  if (n > 0) colnorm_kernel<<<(h + 127) / 128, 128, 0, st>>>(emb, n, h, eps, ahat);
}

long long ee_cross_parts(int max_n, int max_members) {
  const long long t = (max_n + kXT - 1) / kXT;
  return t * t * (max_members + 1);
}

void ee_cross_sumsq(const double* ahat, int n, const double* stored, const int* d_nv, int n_max_stored,
                    long long stride, int m, int h, double* part, double* out, cudaStream_t st) {
  const int tx = (n + kXT - 1) / kXT;
  const int n2 = n_max_stored > n ? n_max_stored : n;
  const int ty = (n2 + kXT - 1) / kXT;
  cross_sumsq_kernel<<<dim3(tx, ty, m + 1), 256, 0, st>>>(ahat, n, stored, d_nv, stride, m, h, part, tx * ty);
  sum_parts_kernel<<<m + 1, 32, 0, st>>>(part, tx * ty, out);
}

void ee_confidence(const float* lp, int n, double* c, cudaStream_t st) {
  confidence_kernel<<<1, 32, 0, st>>>(lp, n, c);
}

void ee_mock_embed(const int* out_tok, long long base, int n, int h, std::uint64_t seed, double* emb,
                   cudaStream_t st) {
  if (n > 0)
    mock_embed_kernel<<<n, h < 256 ? ((h + 31) / 32) * 32 : 256, h * sizeof(double), st>>>(out_tok, base, h,
                                                                                          seed, emb);
}

// hidden-state embedding rows: e[r][c] = x[r][c] / sqrt(mean(x[r]^2) + eps) in
// fp64 from the fp32 final residual rows (the oracle's hidden_embed)
__global__ void hidden_embed_kernel(const float* __restrict__ x, int d, double eps, double* __restrict__ emb) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  double ss = 0.0;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const double v = x[static_cast<long long>(r) * d + c];
    ss = fma(v, v, ss);
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    red[0] = 1.0 / sqrt(t / d + eps);
  }
  __syncthreads();
  const double inv = red[0];
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    emb[static_cast<long long>(r) * d + c] = static_cast<double>(x[static_cast<long long>(r) * d + c]) * inv;
}

void ee_hidden_embed(const float* x, int n, int d, double eps, double* emb, cudaStream_t st) {
  if (n > 0) hidden_embed_kernel<<<n, 256, 0, st>>>(x, d, eps, emb);
}

void ee_corr(const double* emb, int n, int h, double eps, double* gram, double* corr, cudaStream_t st) {
  const long long total = static_cast<long long>(h) * h;
  const int blocks = static_cast<int>((total + 255) / 256 < 592 ? (total + 255) / 256 : 592);
  gram_kernel<<<blocks, 256, 0, st>>>(emb, n, h, gram);
  corr_kernel<<<blocks, 256, 0, st>>>(gram, h, eps, corr);
}

void ee_fcs(const double* corr_new, const double* corrs, int m, int h, double* sim, cudaStream_t st) {
  if (m > 0) fcs_kernel<<<m, 256, 0, st>>>(corr_new, corrs, h, sim);
}


bool ee_fused_mock_supported(int h, int m) { return h <= kEeMaxH && m <= kEeMaxM; }

void ee_fused_mock(const int* out_tok, const float* lp, long long base, int n, int h, std::uint64_t seed, double eps,
                   double* corrs, int m, double* out, cudaStream_t st) {
  const int E = h * (h + 1) / 2;
  const int smem = static_cast<int>((kEeRows * h + h + kEeRows) * sizeof(double) + E * sizeof(std::uint32_t));
  static int attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(ee_fused_mock_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = smem;
  }
  ee_fused_mock_kernel<<<1, kEeThreads, smem, st>>>(out_tok, lp, base, n, h, seed, eps, corrs, m, out);
}

}  // namespace moa::k
