// Agent forward kernels for sm_100a (decode + incremental prefill ticks).
//
// Numerics contract (oracle/model.py mirrors it): bf16 weights and bf16 GEMM
// operands, fp32 accumulation, fp32 residual stream, bf16 KV cache, fp32
// logits.  Every reduction has a fixed order (split-K partials are summed by
// the consumer kernel in slice order), so a tick is bit-reproducible.
#include <cfloat>
#include <climits>
#include <cstdio>

#include "kernels.cuh"

namespace moa::k {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float dot8(uint4 a, uint4 b, float acc) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 u = __bfloat1622float2(x[i]);
    float2 v = __bfloat1622float2(y[i]);
    acc = fmaf(u.x, v.x, acc);
    acc = fmaf(u.y, v.y, acc);
  }
  return acc;
}

// Reduce 32 per-lane values across the warp: afterwards lane L holds the sum
// of value L over all lanes (31 shuffles instead of 32 x 5).
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      float send = upper ? v[i] : v[i + off];
      float keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(kFull, send, off);
    }
  }
  return v[0];
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) s += red[i];
  __syncthreads();
  return s;
}

__device__ __forceinline__ LmStat stat_merge(LmStat a, LmStat b) {
  if (b.s == 0.f) return a;
  if (a.s == 0.f) return b;
  LmStat r;
  if (b.m > a.m || (b.m == a.m && b.idx < a.idx)) {
    r.m = b.m;
    r.idx = b.idx;
  } else {
    r.m = a.m;
    r.idx = a.idx;
  }
  const float da = a.m - r.m, db = b.m - r.m;
  const float ea = __expf(da), eb = __expf(db);
  r.s = ea * a.s + eb * b.s;
  r.t = ea * (a.t + da * a.s) + eb * (b.t + db * b.s);
  return r;
}

// --------------------------------------------------------------------------

__global__ void init_uniform_kernel(bf16* dst, long long n, std::uint64_t base, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    std::uint64_t bits = mix64(base + static_cast<std::uint64_t>(i));
    float u = __fsub_rn(__fmul_rn(static_cast<float>(bits >> 40), 0x1p-23f), 1.0f);
    dst[i] = __float2bfloat16_rn(__fmul_rn(u, scale));
  }
}

__global__ void fill_f32_kernel(float* dst, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = v;
}

__global__ void embed_kernel(const RowDesc* __restrict__ rows, const int* __restrict__ out_tok,
                             const bf16* __restrict__ emb, int d, float* __restrict__ x) {
  const int r = blockIdx.x;
  int t = rows[r].tok;
  if (t < 0) t = out_tok[-1 - t];
  const bf16* e = emb + static_cast<long long>(t) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) x[static_cast<long long>(r) * d + c] = __bfloat162float(e[c]);
}

__global__ void rmsnorm_kernel(const float* __restrict__ x, const int* __restrict__ sel, int d,
                               const float* __restrict__ g, float eps, bf16* __restrict__ h) {
  __shared__ float red[32];
  const int i = blockIdx.x;
  const int r = sel ? sel[i] : i;
  const float* xr = x + static_cast<long long>(r) * d;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) ss = fmaf(xr[c], xr[c], ss);
  ss = block_sum(ss, red);
  const float inv = rsqrtf(ss / static_cast<float>(d) + eps);
  for (int c = threadIdx.x; c < d; c += blockDim.x)
    h[static_cast<long long>(i) * d + c] = __float2bfloat16_rn(xr[c] * inv * g[c]);
}

// Skinny GEMM: each warp owns CPW output columns x RB rows x one K slice.
// Weights stream once per row block through 16-byte non-allocating loads.
constexpr int kRB = 8, kCPW = 4, kWarps = 8;

__global__ void __launch_bounds__(kWarps * 32)
gemm_skinny_kernel(const bf16* __restrict__ A, int R, const bf16* __restrict__ W, int N, int K,
                   int S, float* __restrict__ P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n0 = (blockIdx.x * kWarps + warp) * kCPW;
  const int s = blockIdx.y;
  const int r0 = blockIdx.z * kRB;
  if (n0 >= N) return;
  const int ks = K / S, kb = s * ks, ke = kb + ks;
  const int rows = min(kRB, R - r0);
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  for (int k = kb + lane * 8; k < ke; k += 256) {
    uint4 w[kCPW];
#pragma unroll
    for (int c = 0; c < kCPW; ++c)
      w[c] = (n0 + c < N) ? ldg_stream(W + static_cast<long long>(n0 + c) * K + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int r = 0; r < kRB; ++r) {
      if (r < rows) {
        uint4 a = __ldg(reinterpret_cast<const uint4*>(A + static_cast<long long>(r0 + r) * K + k));
#pragma unroll
        for (int c = 0; c < kCPW; ++c) acc[c * kRB + r] = dot8(a, w[c], acc[c * kRB + r]);
      }
    }
  }
  const float v = transpose_reduce32(acc, lane);
  const int c = lane / kRB, r = lane % kRB;
  if (r < rows && n0 + c < N) P[(static_cast<long long>(s) * R + r0 + r) * N + n0 + c] = v;
}

__global__ void residual_add_kernel(float* __restrict__ x, const float* __restrict__ P, int S,
                                    long long RN) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < RN;
       i += (long long)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < S; ++s) a += P[s * RN + i];
    x[i] += a;
  }
}

__global__ void swiglu_kernel(const float* __restrict__ P, int S, int R, int ffn,
                              bf16* __restrict__ a) {
  const long long total = static_cast<long long>(R) * ffn;
  const long long RN = static_cast<long long>(R) * 2 * ffn;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ffn, j = i % ffn;
    float g = 0.f, u = 0.f;
    for (int s = 0; s < S; ++s) {
      g += P[s * RN + r * 2 * ffn + j];
      u += P[s * RN + r * 2 * ffn + ffn + j];
    }
    const float silu = g / (1.0f + __expf(-g));
    a[i] = __float2bfloat16_rn(silu * u);
  }
}

__global__ void rope_kv_kernel(const float* __restrict__ P, int S, const RowDesc* __restrict__ rows,
                               int R, int nh, int nkv, int hd, const float2* __restrict__ rope,
                               bf16* __restrict__ q, bf16* __restrict__ kpool,
                               bf16* __restrict__ vpool, long long kv_stride, long long layer_off,
                               int max_ctx) {
  const int r = blockIdx.x;
  const RowDesc rd = rows[r];
  const int half = hd / 2;
  const int N = (nh + 2 * nkv) * hd;
  const long long RN = static_cast<long long>(R) * N;
  const float* base = P + static_cast<long long>(r) * N;
  auto get = [&](int c) {
    float a = 0.f;
    for (int s = 0; s < S; ++s) a += base[s * RN + c];
    return a;
  };
  const float2* cs = rope + static_cast<long long>(rd.pos) * half;
  const int pairs = (nh + nkv) * half;
  for (int i = threadIdx.x; i < pairs; i += blockDim.x) {
    const int head = i / half, e = i % half;
    const float x0 = get(head * hd + e), x1 = get(head * hd + e + half);
    const float2 c = cs[e];
    const float y0 = __fsub_rn(__fmul_rn(x0, c.x), __fmul_rn(x1, c.y));
    const float y1 = __fadd_rn(__fmul_rn(x1, c.x), __fmul_rn(x0, c.y));
    if (head < nh) {
      bf16* qo = q + static_cast<long long>(r) * nh * hd + head * hd;
      qo[e] = __float2bfloat16_rn(y0);
      qo[e + half] = __float2bfloat16_rn(y1);
    } else {
      const int kh = head - nh;
      bf16* ko = kpool + rd.kv * kv_stride + layer_off +
                 (static_cast<long long>(kh) * max_ctx + rd.pos) * hd;
      ko[e] = __float2bfloat16_rn(y0);
      ko[e + half] = __float2bfloat16_rn(y1);
    }
  }
  for (int i = threadIdx.x; i < nkv * hd; i += blockDim.x) {
    const int kh = i / hd, e = i % hd;
    bf16* vo = vpool + rd.kv * kv_stride + layer_off +
               (static_cast<long long>(kh) * max_ctx + rd.pos) * hd;
    vo[e] = __float2bfloat16_rn(get((nh + nkv) * hd + i));
  }
}

// One warp per (row, head): online softmax over 32-key blocks.
template <int HD>
__global__ void __launch_bounds__(128)
attention_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, int nh, int nkv,
                 const bf16* __restrict__ kpool, const bf16* __restrict__ vpool,
                 long long kv_stride, long long layer_off, int max_ctx, bf16* __restrict__ o) {
  constexpr int E = HD / 32;
  __shared__ float qs[4][HD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x, h = blockIdx.y * 4 + warp;
  if (h >= nh) return;
  const RowDesc rd = rows[r];
  const int kvh = h / (nh / nkv);
  const bf16* qr = q + (static_cast<long long>(r) * nh + h) * HD;
  for (int e = lane; e < HD; e += 32) qs[warp][e] = __bfloat162float(qr[e]);
  __syncwarp();
  const bf16* K = kpool + rd.kv * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
  const bf16* V = vpool + rd.kv * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
  const float scale = rsqrtf(static_cast<float>(HD));
  float m = -INFINITY, l = 0.f, acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  const int n = rd.pos + 1;
  for (int base = 0; base < n; base += 32) {
    const int j = base + lane;
    float s = -INFINITY;
    if (j < n) {
      const uint4* kp = reinterpret_cast<const uint4*>(K + static_cast<long long>(j) * HD);
      float d = 0.f;
#pragma unroll
      for (int v = 0; v < HD / 8; ++v) {
        uint4 kk = __ldg(kp + v);
        const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kk);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float2 kf = __bfloat1622float2(k2[t]);
          d = fmaf(qs[warp][v * 8 + 2 * t], kf.x, d);
          d = fmaf(qs[warp][v * 8 + 2 * t + 1], kf.y, d);
        }
      }
      s = d * scale;
    }
    float bm = s;
#pragma unroll
    for (int off = 16; off; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, off));
    const float mn = fmaxf(m, bm);
    const float corr = (m == -INFINITY) ? 0.f : __expf(m - mn);
    const float p = (j < n) ? __expf(s - mn) : 0.f;
    float ps = p;
#pragma unroll
    for (int off = 16; off; off >>= 1) ps += __shfl_xor_sync(kFull, ps, off);
    l = l * corr + ps;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] *= corr;
    const int cnt = min(32, n - base);
    for (int jj = 0; jj < cnt; ++jj) {
      const float pj = __shfl_sync(kFull, p, jj);
      const bf16* vr = V + static_cast<long long>(base + jj) * HD + lane * E;
      if constexpr (E == 2) {
        float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        acc[0] = fmaf(pj, vf.x, acc[0]);
        acc[1] = fmaf(pj, vf.y, acc[1]);
      } else {
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr + e));
          acc[e] = fmaf(pj, vf.x, acc[e]);
          acc[e + 1] = fmaf(pj, vf.y, acc[e + 1]);
        }
      }
    }
    m = mn;
  }
  const float inv = 1.0f / l;
  bf16* orow = o + (static_cast<long long>(r) * nh + h) * HD + lane * E;
#pragma unroll
  for (int e = 0; e < E; ++e) orow[e] = __float2bfloat16_rn(acc[e] * inv);
}

// LM head: block b owns a contiguous vocab slice; warps take 4 columns at a
// time for 8 rows; per-lane running stats are merged warp- then block-wide.
constexpr int kLmBlocksPerSm = 4;

__global__ void __launch_bounds__(kWarps * 32)
lm_head_kernel(const bf16* __restrict__ H, int Rl, const bf16* __restrict__ W, int V, int d,
               LmStat* __restrict__ part, float* __restrict__ logits) {
  __shared__ LmStat sm[kWarps][kRB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  const int per = (V + nb - 1) / nb;
  const int c0 = blockIdx.x * per, c1 = min(V, c0 + per);
  for (int r0 = 0; r0 < Rl; r0 += kRB) {
    const int rows = min(kRB, Rl - r0);
    LmStat st{-INFINITY, 0.f, 0.f, INT_MAX};
    for (int cb = c0 + warp * kCPW; cb < c1; cb += kWarps * kCPW) {
      float acc[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.f;
      for (int k = lane * 8; k < d; k += 256) {
        uint4 w[kCPW];
#pragma unroll
        for (int c = 0; c < kCPW; ++c)
          w[c] = (cb + c < c1) ? ldg_stream(W + static_cast<long long>(cb + c) * d + k) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int r = 0; r < kRB; ++r) {
          if (r < rows) {
            uint4 a = __ldg(reinterpret_cast<const uint4*>(H + static_cast<long long>(r0 + r) * d + k));
#pragma unroll
            for (int c = 0; c < kCPW; ++c) acc[c * kRB + r] = dot8(a, w[c], acc[c * kRB + r]);
          }
        }
      }
      const float v = transpose_reduce32(acc, lane);
      const int c = lane / kRB, r = lane % kRB;
      if (r < rows && cb + c < c1) {
        if (logits) logits[static_cast<long long>(r0 + r) * V + cb + c] = v;
        st = stat_merge(st, LmStat{v, 1.f, 0.f, cb + c});
      }
    }
    // lanes r, r+8, r+16, r+24 hold the same row
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) {
      LmStat o{__shfl_xor_sync(kFull, st.m, off), __shfl_xor_sync(kFull, st.s, off),
               __shfl_xor_sync(kFull, st.t, off), __shfl_xor_sync(kFull, st.idx, off)};
      st = (lane & off) ? stat_merge(o, st) : stat_merge(st, o);
    }
    if (lane < kRB) sm[warp][lane] = st;
    __syncthreads();
    if (threadIdx.x < rows) {
      LmStat acc = sm[0][threadIdx.x];
      for (int w = 1; w < kWarps; ++w) acc = stat_merge(acc, sm[w][threadIdx.x]);
      part[static_cast<long long>(r0 + threadIdx.x) * nb + blockIdx.x] = acc;
    }
    __syncthreads();
  }
}

__global__ void lm_merge_kernel(const LmStat* __restrict__ part, int nblk, const int* __restrict__ out_idx,
                                int* __restrict__ out_tok, float* __restrict__ out_lp,
                                float* __restrict__ out_ent) {
  const int r = blockIdx.x, lane = threadIdx.x;
  LmStat st{-INFINITY, 0.f, 0.f, INT_MAX};
  for (int b = lane; b < nblk; b += 32) st = stat_merge(st, part[static_cast<long long>(r) * nblk + b]);
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    LmStat o{__shfl_xor_sync(kFull, st.m, off), __shfl_xor_sync(kFull, st.s, off),
             __shfl_xor_sync(kFull, st.t, off), __shfl_xor_sync(kFull, st.idx, off)};
    st = (lane & off) ? stat_merge(o, st) : stat_merge(st, o);
  }
  if (lane == 0) {
    const int oi = out_idx[r];
    const float ls = logf(st.s);
    out_tok[oi] = st.idx;
    out_lp[oi] = -ls;
    out_ent[oi] = ls - st.t / st.s;
  }
}

inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  return static_cast<int>(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

void init_uniform(bf16* dst, long long n, std::uint64_t base, float scale, cudaStream_t st) {
  init_uniform_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, n, base, scale);
}

void fill_f32(float* dst, long long n, float v, cudaStream_t st) {
  fill_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, n, v);
}

void embed(const RowDesc* rows, int R, const int* out_tok, const bf16* emb, int d, float* x,
           cudaStream_t st) {
  if (R > 0) embed_kernel<<<R, 256, 0, st>>>(rows, out_tok, emb, d, x);
}

void rmsnorm(const float* x, const int* sel, int R, int d, const float* g, float eps, bf16* h,
             cudaStream_t st) {
  if (R > 0) rmsnorm_kernel<<<R, d >= 1024 ? 512 : 256, 0, st>>>(x, sel, d, g, eps, h);
}

void gemm_skinny(const bf16* A, int R, const bf16* W, int N, int K, int S, float* P,
                 cudaStream_t st) {
  if (R <= 0) return;
  dim3 grid((N + kWarps * kCPW - 1) / (kWarps * kCPW), S, (R + kRB - 1) / kRB);
  gemm_skinny_kernel<<<grid, kWarps * 32, 0, st>>>(A, R, W, N, K, S, P);
}

void residual_add(float* x, const float* P, int S, int R, int N, cudaStream_t st) {
  const long long RN = static_cast<long long>(R) * N;
  if (RN > 0) residual_add_kernel<<<grid_for(RN, 256), 256, 0, st>>>(x, P, S, RN);
}

void swiglu(const float* P, int S, int R, int ffn, bf16* a, cudaStream_t st) {
  const long long n = static_cast<long long>(R) * ffn;
  if (n > 0) swiglu_kernel<<<grid_for(n, 256), 256, 0, st>>>(P, S, R, ffn, a);
}

void rope_kv(const float* P, int S, const RowDesc* rows, int R, int nh, int nkv, int hd,
             const float2* rope, bf16* q, bf16* kpool, bf16* vpool, long long kv_stride,
             long long layer_off, int max_ctx, cudaStream_t st) {
  if (R > 0)
    rope_kv_kernel<<<R, 256, 0, st>>>(P, S, rows, R, nh, nkv, hd, rope, q, kpool, vpool, kv_stride,
                                      layer_off, max_ctx);
}

void attention(const bf16* q, const RowDesc* rows, int R, int nh, int nkv, int hd,
               const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off,
               int max_ctx, bf16* o, cudaStream_t st) {
  if (R <= 0) return;
  dim3 grid(R, (nh + 3) / 4);
  if (hd == 64)
    attention_kernel<64><<<grid, 128, 0, st>>>(q, rows, nh, nkv, kpool, vpool, kv_stride, layer_off, max_ctx, o);
  else if (hd == 128)
    attention_kernel<128><<<grid, 128, 0, st>>>(q, rows, nh, nkv, kpool, vpool, kv_stride, layer_off, max_ctx, o);
  else
    printf("attention: unsupported head_dim %d\n", hd);
}

int lm_head_blocks(int V) {
  int nb = 148 * kLmBlocksPerSm;
  return nb < V ? nb : V;
}

void lm_head_stats(const bf16* h, int Rl, const bf16* W, int V, int d, LmStat* part, float* logits,
                   cudaStream_t st) {
  if (Rl > 0) lm_head_kernel<<<lm_head_blocks(V), kWarps * 32, 0, st>>>(h, Rl, W, V, d, part, logits);
}

void lm_merge(const LmStat* part, int Rl, int nblk, const int* out_idx, int* out_tok, float* out_lp,
              float* out_ent, cudaStream_t st) {
  if (Rl > 0) lm_merge_kernel<<<Rl, 32, 0, st>>>(part, nblk, out_idx, out_tok, out_lp, out_ent);
}

}  // namespace moa::k
