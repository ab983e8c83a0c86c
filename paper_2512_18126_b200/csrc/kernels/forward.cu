// Agent forward kernels for sm_100a: decode rows and incremental-prefill rows
// of one tick.
//
// Numerics contract (oracle/model.py mirrors it): bf16 weights and bf16 GEMM
// operands, fp32 accumulation, fp32 residual stream, bf16 KV cache, fp32
// logits.  Every reduction has a fixed order and no tile/split choice depends
// on the batch, so a row's result does not depend on which rows share its
// tick (schedule modes decode identical tokens) and reruns are bit-identical.
#include <cfloat>
#include <climits>
#include <cstdio>
#include <type_traits>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>

#include <cuda.h>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "stamp.cuh"
#include "mma_common.cuh"

namespace moa::k {

// Every forward kernel runs with the maximum shared-memory carveout: when
// consecutive kernels ask for different L1/shared splits the SM must drain
// and reconfigure between them, which serialises the chain and defeats
// programmatic dependent launch.  MOA_CARVEOUT=0 disables (A/B runs).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MOA_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

void uniform_carveout(const void* fn) {
  static std::mutex mu;
  static std::set<const void*> done;
  static const bool on = [] {
    const char* e = std::getenv("MOA_CARVEOUT");
    return !(e && e[0] == '0');
  }();
  if (!on) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert(fn).second) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch: every forward kernel is launched with
// programmatic stream serialisation; it waits for its predecessor's memory
// before touching anything, then immediately lets its successor start
// launching (the successor waits in turn), so launch latency overlaps work.
#define MOA_PDL_ENTRY()                                     \
  do {                                                      \
    asm volatile("griddepcontrol.wait;" ::: "memory");      \
    asm volatile("griddepcontrol.launch_dependents;" :::); \
  } while (0)

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  uniform_carveout(reinterpret_cast<const void*>(kern));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
constexpr int kRB = 8;    // rows per CTA row-block
constexpr int kCPW = 4;   // output columns per warp
constexpr int kWarps = 8;

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

__device__ __forceinline__ void unpack8(uint4 a, float (&f)[8]) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 u = __bfloat1622float2(x[i]);
    f[2 * i] = u.x;
    f[2 * i + 1] = u.y;
  }
}

__device__ __forceinline__ float dot8(const float (&a)[8], uint4 w, float acc) {
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 v = __bfloat1622float2(y[i]);
    acc = fmaf(a[2 * i], v.x, acc);
    acc = fmaf(a[2 * i + 1], v.y, acc);
  }
  return acc;
}

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// Reduce 32 per-lane values across the warp: afterwards lane L holds the sum
// of value L over all lanes (31 shuffles).
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

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// 1 / sqrt(mean(x^2) + eps) of one K-row, computed by one warp in a fixed order.
__device__ __forceinline__ float row_inv_rms(const float* __restrict__ x, int K, float eps, int lane) {
  float ss = 0.f;
  for (int k = lane * 4; k < K; k += 128) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(x + k));
    ss = fmaf(v.x, v.x, ss);
    ss = fmaf(v.y, v.y, ss);
    ss = fmaf(v.z, v.z, ss);
    ss = fmaf(v.w, v.w, ss);
  }
  ss = warp_sum(ss);
  return 1.0f / sqrtf(ss / static_cast<float>(K) + eps);
}

// A fragment: 8 consecutive K elements of one row, as fp32 values of bf16.
template <bool NORM>
__device__ __forceinline__ void load_a(const GemvArgs& a, int row, int k, float (&f)[8]) {
  if constexpr (NORM) {  // normed operand = bf16(x); the row's inverse RMS scales the fp32 result
    const float* x = a.X + static_cast<long long>(row) * a.K + k;
    const float4 x0 = __ldg(reinterpret_cast<const float4*>(x));
    const float4 x1 = __ldg(reinterpret_cast<const float4*>(x + 4));
    f[0] = bf16r(x0.x);
    f[1] = bf16r(x0.y);
    f[2] = bf16r(x0.z);
    f[3] = bf16r(x0.w);
    f[4] = bf16r(x1.x);
    f[5] = bf16r(x1.y);
    f[6] = bf16r(x1.z);
    f[7] = bf16r(x1.w);
  } else {
    unpack8(__ldg(reinterpret_cast<const uint4*>(a.A + static_cast<long long>(row) * a.K + k)), f);
  }
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

__device__ __forceinline__ LmStat shfl_stat(LmStat s, int off) {
  return LmStat{__shfl_xor_sync(kFull, s.m, off), __shfl_xor_sync(kFull, s.s, off),
                __shfl_xor_sync(kFull, s.t, off), __shfl_xor_sync(kFull, s.idx, off)};
}

// --------------------------------------------------------------------------

__global__ void init_uniform_rows_kernel(bf16* dst, long long rows, long long cols, std::uint64_t base,
                                         float scale, int map, int hd) {
  const long long n = rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const std::uint64_t bits = mix64(base + static_cast<std::uint64_t>(i));
    const float u = __fsub_rn(__fmul_rn(static_cast<float>(bits >> 40), 0x1p-23f), 1.0f);
    const long long r = i / cols, c = i % cols;
    long long dr = r;
    if (map == kRowsRopeInterleave) {
      const long long h = r / hd, e = r % hd, half = hd / 2;
      dr = h * hd + (e < half ? 2 * e : 2 * (e - half) + 1);
    } else if (map == kRowsEven) {
      dr = 2 * r;
    } else if (map == kRowsOdd) {
      dr = 2 * r + 1;
    }
    dst[dr * cols + c] = __float2bfloat16_rn(__fmul_rn(u, scale));
  }
}

__global__ void fill_f32_kernel(float* dst, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = v;
}

__global__ void embed_kernel(const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                             const int* __restrict__ out_tok, const bf16* __restrict__ emb, int d,
                             float* __restrict__ x, float* __restrict__ ssq, bf16* __restrict__ xb) {
  MOA_PDL_ENTRY();
  const int r = blockIdx.x;
  if (r >= meta[0]) return;
  int t = rows[r].tok;
  if (t < 0) t = out_tok[-1 - t];
  const bf16* e = emb + static_cast<long long>(t) * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float f[8];
    const uint4 raw = *reinterpret_cast<const uint4*>(e + c);
    unpack8(raw, f);
    if (xb) *reinterpret_cast<uint4*>(xb + static_cast<long long>(r) * d + c) = raw;  // bf16(x): the row itself
    float4* o = reinterpret_cast<float4*>(x + static_cast<long long>(r) * d + c);
    o[0] = make_float4(f[0], f[1], f[2], f[3]);
    o[1] = make_float4(f[4], f[5], f[6], f[7]);
    if (ssq) {  // per-16-column sums of squares (two threads per group) for the next norm
      float sq = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) sq = fmaf(f[i], f[i], sq);
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      if (!(threadIdx.x & 1)) ssq[static_cast<long long>(r) * (d / 16) + c / 16] = sq;
    }
  }
}

// Fused skinny GEMM.  CTA = 8 warps = WG column groups x KP k-parts; a warp
// owns 4 columns x 8 rows x one k-part; k-parts meet in shared memory in a
// fixed order; the epilogue runs on the k-part-0 warps.
template <int WG, bool NORM>
__global__ void __launch_bounds__(kWarps * 32) gemv_kernel(const GemvArgs a) {
  constexpr int KP = kWarps / WG;
  __shared__ float inv_s[kRB];
  __shared__ float red[KP][WG][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = warp % WG, kp = warp / WG;
  const int n0 = (blockIdx.x * WG + cg) * kCPW;
  const int r0 = blockIdx.z * kRB;
  const int kpart = a.K / KP, kb = kp * kpart, ke = kb + kpart;
  // Weights never depend on the previous kernel: the first k-step's weight
  // vectors are in flight before waiting on it (PDL).
  uint4 w_first[kCPW];
#pragma unroll
  for (int c = 0; c < kCPW; ++c)
    w_first[c] = (n0 + c < a.N && kb + lane * 8 < ke)
                     ? ldg_stream(a.W + static_cast<long long>(n0 + c) * a.K + kb + lane * 8)
                     : make_uint4(0, 0, 0, 0);
  const int live = a.meta ? __ldg(a.meta) : a.R;  // tick metadata: not produced by the previous kernel
  // residual of this lane's epilogue element (lane L: column n0 + L/8, row r0 + L%8)
  float res = 0.f;
  if (a.res_early && a.epi == kEpiResidual && kb == 0) {
    const int rr = r0 + lane % kRB, nn = n0 + lane / kRB;
    if (rr < live && nn < a.N) res = a.out[static_cast<long long>(rr) * a.N + nn];
  }
  const unsigned stag = (1u << 16) | (static_cast<unsigned>(a.epi) << 12) | ((a.K >> 4) & 0xfff);
  __shared__ unsigned long long cst[kChainPhases];
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  MOA_PDL_ENTRY();
  if (threadIdx.x == 0) chain_mark(cst, 1);
  if (r0 >= live) return;  // uniform across the CTA
  const int rows = min(kRB, live - r0);
  if constexpr (NORM) {
    if (warp < rows) {
      const float inv = row_inv_rms(a.X + static_cast<long long>(r0 + warp) * a.K, a.K, a.eps, lane);
      if (lane == 0) inv_s[warp] = inv;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) chain_mark(cst, 3);
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = 0.f;
  if (n0 < a.N) {
    for (int k = kb + lane * 8; k < ke; k += 256) {
      uint4 w[kCPW];
#pragma unroll
      for (int c = 0; c < kCPW; ++c)
        w[c] = (k == kb + lane * 8) ? w_first[c]
               : (n0 + c < a.N)     ? ldg_stream(a.W + static_cast<long long>(n0 + c) * a.K + k)
                                    : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int r = 0; r < kRB; ++r) {
        if (r < rows) {
          float f[8];
          load_a<NORM>(a, r0 + r, k, f);
#pragma unroll
          for (int c = 0; c < kCPW; ++c) acc[c * kRB + r] = dot8(f, w[c], acc[c * kRB + r]);
        }
      }
    }
  }
  if (threadIdx.x == 0) chain_mark(cst, 4);
  float v = transpose_reduce32(acc, lane);
  if constexpr (KP > 1) {
    red[kp][cg][lane] = v;
    __syncthreads();
    if (kp != 0) return;
    v = red[0][cg][lane];
#pragma unroll
    for (int p = 1; p < KP; ++p) v += red[p][cg][lane];
  }
  if (threadIdx.x == 0) chain_mark(cst, 5);
  // ---- epilogue: lane L holds column n0 + L/8, row r0 + L%8 ----
  const int c = lane / kRB, r = lane % kRB, n = n0 + c, row = r0 + r;
  const bool ok = r < rows && n < a.N;
  if constexpr (NORM) v *= r < rows ? inv_s[r] : 0.f;  // RMSNorm on the fp32 product
  const float partner = __shfl_xor_sync(kFull, v, kRB);  // column n ^ 1 (same row)
  switch (a.epi) {
    case kEpiF32:
      if (ok) a.out[static_cast<long long>(row) * a.N + n] = v;
      break;
    case kEpiResidual:
      if (ok) {
        float* dst = a.out + static_cast<long long>(row) * a.N + n;
        *dst = (a.res_early ? res : *dst) + v;
      }
      break;
    case kEpiSwiGlu:  // device rows interleave gate (even) / up (odd)
      if (ok && !(n & 1)) {
        const float g = v, u = partner;
        a.out_bf16[static_cast<long long>(row) * (a.N / 2) + n / 2] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
      }
      break;
    case kEpiQkv: {
      if (!ok) break;
      const RowDesc rd = a.rows[row];
      const int hd = a.hd, half = hd / 2;
      const int qk_cols = (a.nh + a.nkv) * hd;
      if (n < qk_cols) {
        if (n & 1) break;  // even lanes own the (x0, x1) RoPE pair
        const int head = n / hd, i = (n % hd) / 2;
        const float2 cs = a.rope[static_cast<long long>(rd.pos) * half + i];
        const float x0 = v, x1 = partner;
        const float y0 = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
        const float y1 = __fadd_rn(__fmul_rn(x1, cs.x), __fmul_rn(x0, cs.y));
        bf16* dst;
        if (head < a.nh) {
          dst = a.out_bf16 + (static_cast<long long>(row) * a.nh + head) * hd;
        } else {
          dst = a.kpool + rd.kv * a.kv_stride + a.layer_off +
                (static_cast<long long>(head - a.nh) * a.max_ctx + rd.pos) * hd;
        }
        dst[i] = __float2bfloat16_rn(y0);
        dst[i + half] = __float2bfloat16_rn(y1);
      } else {
        const int vc = n - qk_cols, kh = vc / hd, e = vc % hd;
        a.vpool[rd.kv * a.kv_stride + a.layer_off + (static_cast<long long>(kh) * a.max_ctx + rd.pos) * hd + e] =
            __float2bfloat16_rn(v);
      }
      break;
    }
  }
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, stag);
  }
}

// Split-KV attention: CTA (row, head, split) covers kv_split(hd) keys with NW
// warps x 32 keys; a row whose context needs several splits writes partials
// and the last CTA to arrive combines them in split order.
template <int HD, int NW>
__global__ void __launch_bounds__(NW * 32)
attention_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta, int nh,
                 int nkv, const bf16* __restrict__ kpool, const bf16* __restrict__ vpool, long long kv_stride,
                 long long layer_off, int max_ctx, bf16* __restrict__ o, float* __restrict__ ws,
                 int* __restrict__ cnt, int nsplit_max) {
  MOA_PDL_ENTRY();
  constexpr int E = HD / 32;
  constexpr int V8 = HD / 8;  // 16-byte vectors per K/V row
  __shared__ float qs[HD];
  __shared__ float wm[NW], wl[NW], wo[NW][HD];
  __shared__ __align__(16) bf16 vs[NW][32][HD];  // V rows of each warp's 32 keys
  __shared__ float ps[NW][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  if (r >= __ldg(meta)) return;
  const RowDesc rd = rows[r];
  const int n = rd.pos + 1;
  const int nsplit = (n + (NW * 32) - 1) / (NW * 32);
  if (s >= nsplit) return;
  const int kvh = h / (nh / nkv);
  const bf16* K = kpool + rd.kv * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
  const bf16* V = vpool + rd.kv * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
  const int base = s * (NW * 32) + warp * 32;
  const int j = base + lane;
  // every lane issues its key's K and V rows at once (2 x HD bf16 in flight)
  uint4 kk[V8], vv[V8];
  if (j < n) {
    const uint4* kp = reinterpret_cast<const uint4*>(K + static_cast<long long>(j) * HD);
    const uint4* vp = reinterpret_cast<const uint4*>(V + static_cast<long long>(j) * HD);
#pragma unroll
    for (int v = 0; v < V8; ++v) kk[v] = __ldg(kp + v);
#pragma unroll
    for (int v = 0; v < V8; ++v) vv[v] = __ldg(vp + v);
  }
  const bf16* qr = q + (static_cast<long long>(r) * nh + h) * HD;
  for (int e = threadIdx.x; e < HD; e += NW * 32) qs[e] = __bfloat162float(qr[e]);
  __syncthreads();
  const float scale = rsqrtf(static_cast<float>(HD));
  float sc = -INFINITY;
  if (j < n) {
    float d = 0.f;
#pragma unroll
    for (int v = 0; v < V8; ++v) {
      float f[8];
      unpack8(kk[v], f);
#pragma unroll
      for (int t = 0; t < 8; ++t) d = fmaf(qs[v * 8 + t], f[t], d);
    }
    sc = d * scale;
    uint4* dst = reinterpret_cast<uint4*>(&vs[warp][lane][0]);
#pragma unroll
    for (int v = 0; v < V8; ++v) dst[v] = vv[v];
  }
  float m = sc;
#pragma unroll
  for (int off = 16; off; off >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, off));
  const float p = (j < n) ? __expf(sc - m) : 0.f;
  const float l = warp_sum(p);
  ps[warp][lane] = p;
  __syncwarp();
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  const int cntk = max(0, min(32, n - base));
  for (int jj = 0; jj < cntk; ++jj) {
    const float pj = ps[warp][jj];
    const bf16* vr = &vs[warp][jj][lane * E];
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      const float2 vf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr + e));
      acc[e] = fmaf(pj, vf.x, acc[e]);
      acc[e + 1] = fmaf(pj, vf.y, acc[e + 1]);
    }
  }
  if (lane == 0) {
    wm[warp] = cntk > 0 ? m : -INFINITY;
    wl[warp] = l;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) wo[warp][lane * E + e] = acc[e];
  __syncthreads();
  // CTA combine of the 4 warps (fixed order)
  float M = wm[0];
  for (int w = 1; w < NW; ++w) M = fmaxf(M, wm[w]);
  float L = 0.f;
  float sw[NW];
  for (int w = 0; w < NW; ++w) {
    sw[w] = wm[w] == -INFINITY ? 0.f : __expf(wm[w] - M);
    L += sw[w] * wl[w];
  }
  bf16* orow = o + (static_cast<long long>(r) * nh + h) * HD;
  if (nsplit == 1) {
    for (int e = threadIdx.x; e < HD; e += NW * 32) {
      float val = 0.f;
      for (int w = 0; w < NW; ++w) val += sw[w] * wo[w][e];
      orow[e] = __float2bfloat16_rn(val / L);
    }
    return;
  }
  float* part = ws + ((static_cast<long long>(r) * nh + h) * nsplit_max + s) * (2 + HD);
  for (int e = threadIdx.x; e < HD; e += NW * 32) {
    float val = 0.f;
    for (int w = 0; w < NW; ++w) val += sw[w] * wo[w][e];
    part[2 + e] = val;
  }
  if (threadIdx.x == 0) {
    part[0] = M;
    part[1] = L;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(cnt + r * nh + h, 1);
    last = prev == nsplit - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const float* pr = ws + (static_cast<long long>(r) * nh + h) * nsplit_max * (2 + HD);
  // split statistics loaded in parallel (thread t: split t), then the
  // weighted sum with every split's partial in flight (fixed split order)
  __shared__ float sw_s[64];
  for (int t = threadIdx.x; t < nsplit; t += NW * 32) sw_s[t] = __ldcg(pr + t * (2 + HD));
  __syncthreads();
  float Mg = -INFINITY;
  for (int t = 0; t < nsplit; ++t) Mg = fmaxf(Mg, sw_s[t]);
  __syncthreads();
  for (int t = threadIdx.x; t < nsplit; t += NW * 32) sw_s[t] = __expf(sw_s[t] - Mg);
  __shared__ float sl_s[64];
  for (int t = threadIdx.x; t < nsplit; t += NW * 32) sl_s[t] = __ldcg(pr + t * (2 + HD) + 1);
  __syncthreads();
  float Lg = 0.f;
  for (int t = 0; t < nsplit; ++t) Lg += sw_s[t] * sl_s[t];
  for (int e = threadIdx.x; e < HD; e += NW * 32) {
    float val = 0.f;
    for (int t0 = 0; t0 < nsplit; t0 += 8) {
      float pv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) pv[u] = t0 + u < nsplit ? __ldcg(pr + (t0 + u) * (2 + HD) + 2 + e) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < nsplit) val += sw_s[t0 + u] * pv[u];
    }
    orow[e] = __float2bfloat16_rn(val / Lg);
  }
  if (threadIdx.x == 0) cnt[r * nh + h] = 0;
}


// GQA attention: CTA = (row, HPG q heads of one kv group, key split of
// kv_split(hd) keys); the CTA's q heads share every K/V load (HPG below the
// group size: more CTAs per row, K/V re-read once per CTA).  Warp w takes 32-key chunks
// w, w+8, ... with an online softmax per head (K: lane = key, full row in
// registers; V: lane = HD/32 output dims of every key), warps combine in
// smem in a fixed order; a row whose context spans several CTAs writes
// per-head partials and the last-arriving CTA combines them in split order.
template <int HD, int HPG>
__global__ void __launch_bounds__(256, 1)
attention_gqa_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta, int nh,
                     int nkv, const bf16* __restrict__ kpool, const bf16* __restrict__ vpool, long long kv_stride,
                     long long layer_off, int max_ctx, bf16* __restrict__ o, float* __restrict__ ws,
                     int* __restrict__ cnt, int nsplit_max, int split_keys, int skip_runs) {
  constexpr int NW = 8, E = HD / 32;
  __shared__ float qs[HPG][HD];
  __shared__ float wm[NW][HPG], wl[NW][HPG];
  __shared__ float wo[NW][HPG][HD];
  __shared__ float cm_s[HPG], cl_s[HPG];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x, s = blockIdx.z;
  const int cpg = (nh / nkv) / HPG;  // CTAs per kv group
  const int g = blockIdx.y / cpg;    // kv head
  const int h0 = g * (nh / nkv) + (blockIdx.y % cpg) * HPG;  // first q head
  // Tick metadata and the keys of earlier ticks are not produced by this
  // forward's previous kernel: read / prefetch them before the PDL wait.
  const int live = __ldg(meta);
  if (r >= live) return;
  const RowDesc rd = rows[r];
  if (skip_runs) {  // rows inside same-agent runs belong to attention_prefill
    if ((r > 0 && rows[r - 1].kv == rd.kv && rows[r - 1].pos + 1 == rd.pos) ||
        (r + 1 < live && rows[r + 1].kv == rd.kv && rows[r + 1].pos == rd.pos + 1))
      return;
  }
  const int n = rd.pos + 1;
  const int nsplit = (n + split_keys - 1) / split_keys;
  if (s >= nsplit) return;
  const int kb = s * split_keys, ke = min(n, kb + split_keys);
  const bf16* K = kpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  const bf16* V = vpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  __shared__ unsigned long long cst[kChainPhases];
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  for (int j = kb + threadIdx.x; j < ke - 1 && j < kb + 2 * NW * 32; j += NW * 32) {  // old keys only (pos is new)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(K + static_cast<long long>(j) * HD));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(V + static_cast<long long>(j) * HD));
  }
  MOA_PDL_ENTRY();
  if (threadIdx.x == 0) chain_mark(cst, 1);
  for (int i = threadIdx.x; i < HPG * HD; i += NW * 32)
    qs[i / HD][i % HD] = __bfloat162float(q[(static_cast<long long>(r) * nh + h0 + i / HD) * HD + i % HD]);
  __syncthreads();
  const float scale = rsqrtf(static_cast<float>(HD));
  float m[HPG], l[HPG], acc[HPG][E];
#pragma unroll
  for (int h = 0; h < HPG; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[h][e] = 0.f;
  }
  // TPK lanes per key (64 dims each): KC keys per warp chunk
  constexpr int TPK = HD / 64, KC = 32 / TPK;
  const int key = lane / TPK, part = lane % TPK;
  using VT = typename std::conditional<E == 2, unsigned, uint2>::type;
  for (int j0 = kb + warp * KC; j0 < ke; j0 += NW * KC) {
    const int j = j0 + key;
    uint4 kk[8];
#pragma unroll
    for (int v = 0; v < 8; ++v)
      kk[v] = j < ke ? __ldg(reinterpret_cast<const uint4*>(K + static_cast<long long>(j) * HD + part * 64) + v)
                     : make_uint4(0, 0, 0, 0);
    VT vv[KC];
#pragma unroll
    for (int jj = 0; jj < KC; ++jj)
      vv[jj] = j0 + jj < ke ? __ldg(reinterpret_cast<const VT*>(V + static_cast<long long>(j0 + jj) * HD + lane * E)) : VT{};
#pragma unroll
    for (int h = 0; h < HPG; ++h) {
      float dv[8];  // one partial per 16-byte chunk: 8 short FMA chains instead of one of 64
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        float f[8];
        unpack8(kk[v], f);
        dv[v] = 0.f;
#pragma unroll
        for (int t = 0; t < 8; ++t) dv[v] = fmaf(qs[h][part * 64 + v * 8 + t], f[t], dv[v]);
      }
      float d = ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
      if constexpr (TPK == 2) d += __shfl_xor_sync(kFull, d, 1);
      const float sc = j < ke ? d * scale : -INFINITY;
      float cmax = sc;
#pragma unroll
      for (int off = 16; off; off >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(kFull, cmax, off));
      const float mn = fmaxf(m[h], cmax);
      const float resc = m[h] == -INFINITY ? 0.f : __expf(m[h] - mn);
      const float p = j < ke ? __expf(sc - mn) : 0.f;
      l[h] = l[h] * resc + warp_sum(part == 0 ? p : 0.f);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[h][e] *= resc;
#pragma unroll
      for (int jj = 0; jj < KC; ++jj) {
        const float pj = __shfl_sync(kFull, p, jj * TPK);
        if constexpr (E == 2) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj]));
          acc[h][0] = fmaf(pj, f.x, acc[h][0]);
          acc[h][1] = fmaf(pj, f.y, acc[h][1]);
        } else {
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].x));
          const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].y));
          acc[h][0] = fmaf(pj, f0.x, acc[h][0]);
          acc[h][1] = fmaf(pj, f0.y, acc[h][1]);
          acc[h][2] = fmaf(pj, f1.x, acc[h][2]);
          acc[h][3] = fmaf(pj, f1.y, acc[h][3]);
        }
      }
      m[h] = mn;
    }
  }
#pragma unroll
  for (int h = 0; h < HPG; ++h) {
    if (lane == 0) {
      wm[warp][h] = m[h];
      wl[warp][h] = l[h];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) wo[warp][h][lane * E + e] = acc[h][e];
  }
  __syncthreads();
  // CTA combine of the warps, per head, fixed warp order
  if (threadIdx.x < HPG) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w][h]);
    float Lsum = 0.f;
    for (int w = 0; w < NW; ++w) Lsum += wm[w][h] == -INFINITY ? 0.f : __expf(wm[w][h] - M) * wl[w][h];
    cm_s[h] = M;
    cl_s[h] = Lsum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HPG * HD; i += NW * 32) {
    const int h = i / HD, e = i % HD;
    const float M = cm_s[h];
    float val = 0.f;
    for (int w = 0; w < NW; ++w)
      if (wm[w][h] != -INFINITY) val += __expf(wm[w][h] - M) * wo[w][h][e];
    const int head = h0 + h;
    if (nsplit == 1) {
      o[(static_cast<long long>(r) * nh + head) * HD + e] = __float2bfloat16_rn(val / cl_s[h]);
    } else {
      float* part = ws + ((static_cast<long long>(r) * nh + head) * nsplit_max + s) * (2 + HD);
      __stcg(part + 2 + e, val);
      if (e == 0) {
        __stcg(part, M);
        __stcg(part + 1, cl_s[h]);
      }
    }
  }
  if (nsplit == 1) {
    if (threadIdx.x == 0) {
      chain_mark(cst, 2);
      chain_flush(cst, 6u << 16);
    }
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                 : "=r"(prev)
                 : "l"(cnt + r * gridDim.y + blockIdx.y)
                 : "memory");
    last = prev == static_cast<unsigned>(nsplit - 1);
  }
  __syncthreads();
  if (!last) return;
  // combine the splits (split order); split stats read in parallel
  __shared__ float sw_s[HPG][64];
  for (int i = threadIdx.x; i < HPG * nsplit; i += NW * 32) {
    const int h = i / nsplit, t = i % nsplit;
    sw_s[h][t] = __ldcg(ws + ((static_cast<long long>(r) * nh + h0 + h) * nsplit_max + t) * (2 + HD));
  }
  __syncthreads();
  if (threadIdx.x < HPG) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int t = 0; t < nsplit; ++t) M = fmaxf(M, sw_s[h][t]);
    float Lsum = 0.f;
    for (int t = 0; t < nsplit; ++t) {
      const float w = __expf(sw_s[h][t] - M);
      Lsum += w * __ldcg(ws + ((static_cast<long long>(r) * nh + h0 + h) * nsplit_max + t) * (2 + HD) + 1);
      sw_s[h][t] = w;
    }
    cl_s[h] = Lsum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < HPG * HD; i += NW * 32) {
    const int h = i / HD, e = i % HD;
    const float* pr = ws + (static_cast<long long>(r) * nh + h0 + h) * nsplit_max * (2 + HD);
    float val = 0.f;
    for (int t0 = 0; t0 < nsplit; t0 += 8) {
      float pv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) pv[u] = t0 + u < nsplit ? __ldcg(pr + (t0 + u) * (2 + HD) + 2 + e) : 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (t0 + u < nsplit) val += sw_s[h][t0 + u] * pv[u];
    }
    o[(static_cast<long long>(r) * nh + h0 + h) * HD + e] = __float2bfloat16_rn(val / cl_s[h]);
  }
  if (threadIdx.x == 0) cnt[r * gridDim.y + blockIdx.y] = 0;
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, 6u << 16);
  }
}


// Prefill attention: CTA = (64 consecutive rows of the tick, q head), 8 warps
// x 8 rows.  The rows of one agent's prefill job are consecutive with
// increasing positions, so the block's rows split into a few same-agent
// segments; for each, the segment's keys stream through smem in blocks of
// 64 (K transposed, fp32) shared by every row of the segment, each warp runs
// an online softmax for its rows (lane = 2 keys for the scores, lane = HD/32
// output dims for P.V) with the causal mask pos(key) <= pos(row).  Replaces
// one CTA per (row, kv head) re-reading the whole context from L2 for every
// row of a long prompt.
constexpr int kPfRows = 64, kPfKeys = 64;
template <int HD>
__global__ void __launch_bounds__(256, 1)
attention_prefill_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                         int nh, int nkv, const bf16* __restrict__ kpool, const bf16* __restrict__ vpool,
                         long long kv_stride, long long layer_off, int max_ctx, bf16* __restrict__ o) {
  constexpr int E = HD / 32, KS = kPfKeys + 1;  // Kt row stride (fp32): conflict-free transposed stores
  extern __shared__ __align__(16) float pf_sm[];
  float* Kt = pf_sm;                       // [HD][KS]
  float* Vs = Kt + HD * KS;                // [64][HD]
  float* Qs = Vs + kPfKeys * HD;           // [8 warps][8 rows][HD]
  float* Ps = Qs + 8 * 8 * HD;             // [8 warps][64 keys][8 rows]
  __shared__ int seg_s[kPfRows + 1], seg_end_s[kPfRows];
  __shared__ int nseg_s;
  __shared__ RowDesc rd_s[kPfRows];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = blockIdx.x * kPfRows, h = blockIdx.y;
  const int live = __ldg(meta);
  if (b0 >= live) return;
  const int nb = min(kPfRows, live - b0);
  const int g = h / (nh / nkv);
  if (threadIdx.x < nb) rd_s[threadIdx.x] = rows[b0 + threadIdx.x];  // tick metadata (not the previous kernel's)
  __syncthreads();
  if (threadIdx.x == 0) {
    // same-agent runs of consecutive positions; a row alone in its run (a
    // decode row) is left to the per-row kernel (attention(..., skip_runs))
    int n = 0;
    for (int i = 0; i < nb; ++i)
      if (i == 0 || rd_s[i].kv != rd_s[i - 1].kv || rd_s[i].pos != rd_s[i - 1].pos + 1) seg_s[n++] = i;
    seg_s[n] = nb;
    int m = 0;
    for (int k = 0; k < n; ++k) {
      const int a = seg_s[k], b = seg_s[k + 1];
      const bool single = b - a == 1 && !(a == 0 && b0 > 0 && rows[b0 - 1].kv == rd_s[0].kv &&
                                            rows[b0 - 1].pos + 1 == rd_s[0].pos) &&
                          !(b == nb && b0 + nb < live && rows[b0 + nb].kv == rd_s[nb - 1].kv &&
                            rows[b0 + nb].pos == rd_s[nb - 1].pos + 1);
      if (!single) {
        seg_s[m] = a;
        seg_end_s[m] = b;
        ++m;
      }
    }
    nseg_s = m;
  }
  MOA_PDL_ENTRY();
  __syncthreads();
  const float scale = rsqrtf(static_cast<float>(HD));
  float* qs = Qs + warp * 8 * HD;
  float* ps = Ps + warp * kPfKeys * 8;
  for (int sg = 0; sg < nseg_s; ++sg) {
    const int a = seg_s[sg], b = seg_end_s[sg];
    const RowDesc first = rd_s[a];
    const int maxpos = rd_s[b - 1].pos;
    const bf16* K = kpool + first.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
    const bf16* V = vpool + first.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
    // this warp's rows of the segment: block rows [warp*8, warp*8+8) within [a, b)
    const int r_lo = max(a, warp * 8), r_hi = min(b, warp * 8 + 8);
    const bool active = r_lo < r_hi;
    int pos[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) pos[r] = (warp * 8 + r >= r_lo && warp * 8 + r < r_hi) ? rd_s[warp * 8 + r].pos : -1;
    if (active)
      for (int i = lane; i < 8 * HD; i += 32) {
        const int r = i / HD, d = i % HD;
        qs[i] = pos[r] >= 0 ? __bfloat162float(q[(static_cast<long long>(b0 + warp * 8 + r) * nh + h) * HD + d]) : 0.f;
      }
    float m[8], l[8], acc[8][E];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      m[r] = -INFINITY;
      l[r] = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[r][e] = 0.f;
    }
    for (int kb = 0; kb <= maxpos; kb += kPfKeys) {
      __syncthreads();  // the previous key block is consumed
      for (int c = threadIdx.x; c < kPfKeys * (HD / 8); c += 256) {
        const int key = c / (HD / 8), d0 = (c % (HD / 8)) * 8;
        float kf[8], vf[8];
        if (kb + key <= maxpos) {
          unpack8(__ldcg(reinterpret_cast<const uint4*>(K + static_cast<long long>(kb + key) * HD + d0)), kf);
          unpack8(__ldcg(reinterpret_cast<const uint4*>(V + static_cast<long long>(kb + key) * HD + d0)), vf);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) kf[i] = vf[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) Kt[(d0 + i) * KS + key] = kf[i];
        *reinterpret_cast<float4*>(Vs + key * HD + d0) = make_float4(vf[0], vf[1], vf[2], vf[3]);
        *reinterpret_cast<float4*>(Vs + key * HD + d0 + 4) = make_float4(vf[4], vf[5], vf[6], vf[7]);
      }
      __syncthreads();
      if (!active) continue;
      float s0[8], s1[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) s0[r] = s1[r] = 0.f;
      for (int d = 0; d < HD; d += 4) {
        float k0[4], k1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          k0[i] = Kt[(d + i) * KS + lane];
          k1[i] = Kt[(d + i) * KS + lane + 32];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float4 qv = *reinterpret_cast<const float4*>(qs + r * HD + d);
          s0[r] = fmaf(qv.x, k0[0], fmaf(qv.y, k0[1], fmaf(qv.z, k0[2], fmaf(qv.w, k0[3], s0[r]))));
          s1[r] = fmaf(qv.x, k1[0], fmaf(qv.y, k1[1], fmaf(qv.z, k1[2], fmaf(qv.w, k1[3], s1[r]))));
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const bool ok0 = kb + lane <= pos[r], ok1 = kb + lane + 32 <= pos[r];
        const float a0 = ok0 ? s0[r] * scale : -INFINITY, a1 = ok1 ? s1[r] * scale : -INFINITY;
        float bm = fmaxf(a0, a1);
#pragma unroll
        for (int off = 16; off; off >>= 1) bm = fmaxf(bm, __shfl_xor_sync(kFull, bm, off));
        const float mn = fmaxf(m[r], bm);
        const float corr = (m[r] == -INFINITY) ? 0.f : __expf(m[r] - mn);
        const float p0 = ok0 ? __expf(a0 - mn) : 0.f, p1 = ok1 ? __expf(a1 - mn) : 0.f;
        if (mn != -INFINITY) {  // rows with no key in this block keep their state
          l[r] = l[r] * corr + warp_sum(p0 + p1);
#pragma unroll
          for (int e = 0; e < E; ++e) acc[r][e] *= corr;
          m[r] = mn;
        }
        ps[lane * 8 + r] = p0;
        ps[(lane + 32) * 8 + r] = p1;
      }
      __syncwarp();
      for (int k = 0; k < kPfKeys && kb + k <= maxpos; ++k) {
        const float4 pa = *reinterpret_cast<const float4*>(ps + k * 8);
        const float4 pb = *reinterpret_cast<const float4*>(ps + k * 8 + 4);
        const float pk[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const float v = Vs[k * HD + lane + 32 * e];
#pragma unroll
          for (int r = 0; r < 8; ++r) acc[r][e] = fmaf(pk[r], v, acc[r][e]);
        }
      }
      __syncwarp();
    }
    if (active) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (pos[r] < 0) continue;
        const float inv = 1.0f / l[r];
#pragma unroll
        for (int e = 0; e < E; ++e)
          o[(static_cast<long long>(b0 + warp * 8 + r) * nh + h) * HD + lane + 32 * e] = __float2bfloat16_rn(acc[r][e] * inv);
      }
    }
  }
}

// Prefill attention on the tensor cores (mma.sync m16n8k16 bf16 -> fp32,
// FlashAttention-2 dataflow): CTA = (64 consecutive rows of the tick, q head),
// 4 warps x 16 rows.  Same segment logic as attention_prefill_kernel (rows
// alone in their run are left to the per-row kernel).  Per segment the Q rows
// stay in registers as A fragments; each 64-key block of K and V is staged in
// smem (16-byte chunks XOR-swizzled by row so ldmatrix is conflict-free);
// S = Q.K^T per warp (8 n-tiles), causal mask by position, online softmax on
// the accumulator fragments, P reused in registers as the A operand of P.V.
template <int HD>
__global__ void __launch_bounds__(128, 1)
attention_prefill_mma_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                             int nh, int nkv, const bf16* __restrict__ kpool, const bf16* __restrict__ vpool,
                             long long kv_stride, long long layer_off, int max_ctx, bf16* __restrict__ o) {
  constexpr int RB = HD * 2;       // smem row bytes
  constexpr int KSTEPS = HD / 16;  // k-steps of Q.K^T
  constexpr int NT = HD / 8;       // n-tiles of P.V
  extern __shared__ __align__(128) unsigned char pm_sm[];
  unsigned char* Qs = pm_sm;                 // [64][HD] bf16, swizzled
  unsigned char* Ks = Qs + kPfRows * RB;     // [64][HD]
  unsigned char* Vs = Ks + kPfKeys * RB;     // [64][HD]
  __shared__ int seg_s[kPfRows + 1], seg_end_s[kPfRows];
  __shared__ int nseg_s;
  __shared__ RowDesc rd_s[kPfRows];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int b0 = blockIdx.x * kPfRows, h = blockIdx.y;
  const int live = __ldg(meta);
  if (b0 >= live) return;
  const int nb = min(kPfRows, live - b0);
  const int kvh = h / (nh / nkv);
  if (threadIdx.x < nb) rd_s[threadIdx.x] = rows[b0 + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int i = 0; i < nb; ++i)
      if (i == 0 || rd_s[i].kv != rd_s[i - 1].kv || rd_s[i].pos != rd_s[i - 1].pos + 1) seg_s[n++] = i;
    seg_s[n] = nb;
    int m = 0;
    for (int k = 0; k < n; ++k) {
      const int a = seg_s[k], b = seg_s[k + 1];
      const bool single = b - a == 1 && !(a == 0 && b0 > 0 && rows[b0 - 1].kv == rd_s[0].kv &&
                                            rows[b0 - 1].pos + 1 == rd_s[0].pos) &&
                          !(b == nb && b0 + nb < live && rows[b0 + nb].kv == rd_s[nb - 1].kv &&
                            rows[b0 + nb].pos == rd_s[nb - 1].pos + 1);
      if (!single) {
        seg_s[m] = a;
        seg_end_s[m] = b;
        ++m;
      }
    }
    nseg_s = m;
  }
  MOA_PDL_ENTRY();
  // Q rows of the block -> smem (rows past the live ones: zeros)
  for (int c = threadIdx.x; c < kPfRows * (HD / 8); c += 128) {
    const int r = c / (HD / 8), ch = c % (HD / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < nb) v = __ldcg(reinterpret_cast<const uint4*>(q + (static_cast<long long>(b0 + r) * nh + h) * HD) + ch);
    *reinterpret_cast<uint4*>(Qs + r * RB + ((ch ^ (r & 7)) << 4)) = v;
  }
  __syncthreads();
  const std::uint32_t qs_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Qs));
  const std::uint32_t ks_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Ks));
  const std::uint32_t vs_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Vs));
  // A fragments of this warp's 16 rows
  std::uint32_t qa[KSTEPS][4];
  {
    const int r = warp * 16 + (lane & 15);
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int ch = kk * 2 + (lane >> 4);
      ldsm_x4(qs_u + r * RB + ((ch ^ (r & 7)) << 4), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
    }
  }
  const float sl2 = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;  // scale * log2(e)
  const int ra = warp * 16 + g8, rb = ra + 8;  // block rows of this thread's two accumulator rows
  for (int sg = 0; sg < nseg_s; ++sg) {
    const int a = seg_s[sg], b = seg_end_s[sg];
    const int maxpos = rd_s[b - 1].pos;
    const int kvslot = rd_s[a].kv;
    const bf16* K = kpool + kvslot * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
    const bf16* V = vpool + kvslot * kv_stride + layer_off + static_cast<long long>(kvh) * max_ctx * HD;
    const int pa = (ra >= a && ra < b) ? rd_s[ra].pos : -1, pb = (rb >= a && rb < b) ? rd_s[rb].pos : -1;
    const bool warp_active = warp * 16 < b && warp * 16 + 16 > a;
    float m_a = -1e30f, m_b = -1e30f, l_a = 0.f, l_b = 0.f;
    float oacc[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) oacc[nt][0] = oacc[nt][1] = oacc[nt][2] = oacc[nt][3] = 0.f;
    for (int kb = 0; kb <= maxpos; kb += kPfKeys) {
      __syncthreads();  // the previous block's K / V are consumed
      for (int c = threadIdx.x; c < kPfKeys * (HD / 8); c += 128) {
        const int r = c / (HD / 8), ch = c % (HD / 8);
        uint4 kv4 = make_uint4(0, 0, 0, 0), vv4 = make_uint4(0, 0, 0, 0);
        if (kb + r <= maxpos) {
          kv4 = __ldcg(reinterpret_cast<const uint4*>(K + static_cast<long long>(kb + r) * HD) + ch);
          vv4 = __ldcg(reinterpret_cast<const uint4*>(V + static_cast<long long>(kb + r) * HD) + ch);
        }
        *reinterpret_cast<uint4*>(Ks + r * RB + ((ch ^ (r & 7)) << 4)) = kv4;
        *reinterpret_cast<uint4*>(Vs + r * RB + ((ch ^ (r & 7)) << 4)) = vv4;
      }
      __syncthreads();
      if (!warp_active) continue;
      // S = Q K^T: 16 rows x 64 keys (8 n-tiles of 8 keys)
      float sacc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {  // two n-tiles per ldmatrix.x4
          const int kr = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = kk * 2 + ((lane >> 3) & 1);
          std::uint32_t b00, b01, b10, b11;
          ldsm_x4(ks_u + kr * RB + ((ch ^ (kr & 7)) << 4), b00, b01, b10, b11);
          mma_bf16(sacc[2 * jp], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b00, b01);
          mma_bf16(sacc[2 * jp + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b10, b11);
        }
      }
      // causal mask + online softmax (rows ra: c0,c1; rb: c2,c3), in log2 units
      float mx_a = -1e30f, mx_b = -1e30f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int key = kb + 8 * j + 2 * t4;
        sacc[j][0] = key <= pa ? sacc[j][0] * sl2 : -1e30f;
        sacc[j][1] = key + 1 <= pa ? sacc[j][1] * sl2 : -1e30f;
        sacc[j][2] = key <= pb ? sacc[j][2] * sl2 : -1e30f;
        sacc[j][3] = key + 1 <= pb ? sacc[j][3] * sl2 : -1e30f;
        mx_a = fmaxf(mx_a, fmaxf(sacc[j][0], sacc[j][1]));
        mx_b = fmaxf(mx_b, fmaxf(sacc[j][2], sacc[j][3]));
      }
      mx_a = fmaxf(mx_a, __shfl_xor_sync(kFull, mx_a, 1));
      mx_a = fmaxf(mx_a, __shfl_xor_sync(kFull, mx_a, 2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(kFull, mx_b, 1));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(kFull, mx_b, 2));
      const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
      const float ca = exp2f(m_a - mn_a), cb = exp2f(m_b - mn_b);
      m_a = mn_a;
      m_b = mn_b;
      float ps_a = 0.f, ps_b = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sacc[j][0] = sacc[j][0] <= -1e29f ? 0.f : exp2f(sacc[j][0] - mn_a);
        sacc[j][1] = sacc[j][1] <= -1e29f ? 0.f : exp2f(sacc[j][1] - mn_a);
        sacc[j][2] = sacc[j][2] <= -1e29f ? 0.f : exp2f(sacc[j][2] - mn_b);
        sacc[j][3] = sacc[j][3] <= -1e29f ? 0.f : exp2f(sacc[j][3] - mn_b);
        ps_a += sacc[j][0] + sacc[j][1];
        ps_b += sacc[j][2] + sacc[j][3];
      }
      l_a = l_a * ca + ps_a;
      l_b = l_b * cb + ps_b;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        oacc[nt][0] *= ca;
        oacc[nt][1] *= ca;
        oacc[nt][2] *= cb;
        oacc[nt][3] *= cb;
      }
      // O += P V: P (16 x 64) from the S fragments, V^T fragments by ldmatrix.trans
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const std::uint32_t pa0 = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
        const std::uint32_t pa1 = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
        const std::uint32_t pa2 = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
        const std::uint32_t pa3 = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
        for (int np = 0; np < NT / 2; ++np) {  // two dim n-tiles per ldmatrix.x4.trans
          const int vr = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int ch = np * 2 + (lane >> 4);
          std::uint32_t v00, v01, v10, v11;
          ldsm_x4_t(vs_u + vr * RB + ((ch ^ (vr & 7)) << 4), v00, v01, v10, v11);
          mma_bf16(oacc[2 * np], pa0, pa1, pa2, pa3, v00, v01);
          mma_bf16(oacc[2 * np + 1], pa0, pa1, pa2, pa3, v10, v11);
        }
      }
    }
    if (warp_active) {
      l_a += __shfl_xor_sync(kFull, l_a, 1);
      l_a += __shfl_xor_sync(kFull, l_a, 2);
      l_b += __shfl_xor_sync(kFull, l_b, 1);
      l_b += __shfl_xor_sync(kFull, l_b, 2);
      const float ia = pa >= 0 ? 1.0f / l_a : 0.f, ib = pb >= 0 ? 1.0f / l_b : 0.f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int d = nt * 8 + 2 * t4;
        if (pa >= 0)
          *reinterpret_cast<__nv_bfloat162*>(o + (static_cast<long long>(b0 + ra) * nh + h) * HD + d) =
              __floats2bfloat162_rn(oacc[nt][0] * ia, oacc[nt][1] * ia);
        if (pb >= 0)
          *reinterpret_cast<__nv_bfloat162*>(o + (static_cast<long long>(b0 + rb) * nh + h) * HD + d) =
              __floats2bfloat162_rn(oacc[nt][2] * ib, oacc[nt][3] * ib);
      }
    }
  }
}

// GQA decode attention on the tensor cores: CTA = (row, kv head, key split),
// 4 warps.  The group's q heads (<= 16) are the M rows of an m16n8k16 tile
// (rows past the group are zero), so one K/V read serves every head of the
// group at MMA speed.  Warp w takes the split's 64-key blocks w, w+4, ...: it
// stages K and V of a block in its own swizzled smem slice, S = Q.K^T,
// online softmax on the fragments, O += P.V; the warps then combine in smem
// in a fixed order and a row spanning several splits is combined by the
// last-arriving CTA (as attention_gqa_kernel).
template <int HD>
__global__ void __launch_bounds__(128, 1)
attention_decode_mma_kernel(const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                            int nh, int nkv, const bf16* __restrict__ kpool, const bf16* __restrict__ vpool,
                            long long kv_stride, long long layer_off, int max_ctx, bf16* __restrict__ o,
                            float* __restrict__ ws, int* __restrict__ cnt, int nsplit_max, int split_keys,
                            int skip_runs) {
  constexpr int RB = HD * 2, KSTEPS = HD / 16, NT = HD / 8, NWARP = 4;
  extern __shared__ __align__(128) unsigned char dm_sm[];
  unsigned char* Qs = dm_sm;                           // [16][HD] bf16, swizzled
  unsigned char* KV = dm_sm + 16 * RB;                 // per warp: K [64][HD], V [64][HD]
  float* wo = reinterpret_cast<float*>(KV);            // after the key loop: [4 warps][16][HD] fp32
  __shared__ float wm[NWARP][16], wl[NWARP][16], cm_s[16], cl_s[16];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int r = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int live = __ldg(meta);
  if (r >= live) return;
  const RowDesc rd = rows[r];
  if (skip_runs) {
    if ((r > 0 && rows[r - 1].kv == rd.kv && rows[r - 1].pos + 1 == rd.pos) ||
        (r + 1 < live && rows[r + 1].kv == rd.kv && rows[r + 1].pos == rd.pos + 1))
      return;
  }
  const int n = rd.pos + 1;
  const int nsplit = (n + split_keys - 1) / split_keys;
  if (s >= nsplit) return;
  const int hpg = nh / nkv;
  const int kb = s * split_keys, ke = min(n, kb + split_keys);
  const bf16* K = kpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  const bf16* V = vpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  for (int j = kb + threadIdx.x; j < ke - 1 && j < kb + 4 * 128; j += 128) {  // old keys only (pos is new)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(K + static_cast<long long>(j) * HD));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(V + static_cast<long long>(j) * HD));
  }
  MOA_PDL_ENTRY();
  for (int c = threadIdx.x; c < 16 * (HD / 8); c += 128) {
    const int hr = c / (HD / 8), ch = c % (HD / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (hr < hpg) v = __ldcg(reinterpret_cast<const uint4*>(q + (static_cast<long long>(r) * nh + g * hpg + hr) * HD) + ch);
    *reinterpret_cast<uint4*>(Qs + hr * RB + ((ch ^ (hr & 7)) << 4)) = v;
  }
  __syncthreads();
  const std::uint32_t qs_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Qs));
  unsigned char* Ks = KV + warp * 2 * kPfKeys * RB;
  unsigned char* Vs = Ks + kPfKeys * RB;
  const std::uint32_t ks_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Ks));
  const std::uint32_t vs_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Vs));
  std::uint32_t qa[KSTEPS][4];
#pragma unroll
  for (int kk = 0; kk < KSTEPS; ++kk) {
    const int hr = lane & 15, ch = kk * 2 + (lane >> 4);
    ldsm_x4(qs_u + hr * RB + ((ch ^ (hr & 7)) << 4), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
  }
  const float sl2 = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;
  float m_a = -1e30f, m_b = -1e30f, l_a = 0.f, l_b = 0.f;
  float oacc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) oacc[nt][0] = oacc[nt][1] = oacc[nt][2] = oacc[nt][3] = 0.f;
  for (int b0k = kb + warp * kPfKeys; b0k < ke; b0k += NWARP * kPfKeys) {
    // stage this warp's block (all loads in flight, then the stores)
    constexpr int CH = kPfKeys * (HD / 8) / 32;  // 16-byte chunks per lane per matrix
#pragma unroll
    for (int i0 = 0; i0 < CH; i0 += 8) {  // 8 K + 8 V chunks in flight per lane
      uint4 kr[8], vr[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = (i0 + i) * 32 + lane, key = c / (HD / 8), ch = c % (HD / 8);
        const bool ok = b0k + key < ke;
        kr[i] = ok ? __ldcg(reinterpret_cast<const uint4*>(K + static_cast<long long>(b0k + key) * HD) + ch)
                   : make_uint4(0, 0, 0, 0);
        vr[i] = ok ? __ldcg(reinterpret_cast<const uint4*>(V + static_cast<long long>(b0k + key) * HD) + ch)
                   : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int c = (i0 + i) * 32 + lane, key = c / (HD / 8), ch = c % (HD / 8);
        *reinterpret_cast<uint4*>(Ks + key * RB + ((ch ^ (key & 7)) << 4)) = kr[i];
        *reinterpret_cast<uint4*>(Vs + key * RB + ((ch ^ (key & 7)) << 4)) = vr[i];
      }
    }
    __syncwarp();
    float sacc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        const int krow = jp * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        std::uint32_t b00, b01, b10, b11;
        ldsm_x4(ks_u + krow * RB + ((ch ^ (krow & 7)) << 4), b00, b01, b10, b11);
        mma_bf16(sacc[2 * jp], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b00, b01);
        mma_bf16(sacc[2 * jp + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b10, b11);
      }
    }
    float mx_a = -1e30f, mx_b = -1e30f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int key = b0k + 8 * j + 2 * t4;
      sacc[j][0] = key < ke ? sacc[j][0] * sl2 : -1e30f;
      sacc[j][1] = key + 1 < ke ? sacc[j][1] * sl2 : -1e30f;
      sacc[j][2] = key < ke ? sacc[j][2] * sl2 : -1e30f;
      sacc[j][3] = key + 1 < ke ? sacc[j][3] * sl2 : -1e30f;
      mx_a = fmaxf(mx_a, fmaxf(sacc[j][0], sacc[j][1]));
      mx_b = fmaxf(mx_b, fmaxf(sacc[j][2], sacc[j][3]));
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(kFull, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(kFull, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(kFull, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(kFull, mx_b, 2));
    const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
    const float ca = exp2f(m_a - mn_a), cb = exp2f(m_b - mn_b);
    m_a = mn_a;
    m_b = mn_b;
    float ps_a = 0.f, ps_b = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      sacc[j][0] = sacc[j][0] <= -1e29f ? 0.f : exp2f(sacc[j][0] - mn_a);
      sacc[j][1] = sacc[j][1] <= -1e29f ? 0.f : exp2f(sacc[j][1] - mn_a);
      sacc[j][2] = sacc[j][2] <= -1e29f ? 0.f : exp2f(sacc[j][2] - mn_b);
      sacc[j][3] = sacc[j][3] <= -1e29f ? 0.f : exp2f(sacc[j][3] - mn_b);
      ps_a += sacc[j][0] + sacc[j][1];
      ps_b += sacc[j][2] + sacc[j][3];
    }
    l_a = l_a * ca + ps_a;
    l_b = l_b * cb + ps_b;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      oacc[nt][0] *= ca;
      oacc[nt][1] *= ca;
      oacc[nt][2] *= cb;
      oacc[nt][3] *= cb;
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const std::uint32_t pa0 = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
      const std::uint32_t pa1 = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
      const std::uint32_t pa2 = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
      const std::uint32_t pa3 = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int vrow = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = np * 2 + (lane >> 4);
        std::uint32_t v00, v01, v10, v11;
        ldsm_x4_t(vs_u + vrow * RB + ((ch ^ (vrow & 7)) << 4), v00, v01, v10, v11);
        mma_bf16(oacc[2 * np], pa0, pa1, pa2, pa3, v00, v01);
        mma_bf16(oacc[2 * np + 1], pa0, pa1, pa2, pa3, v10, v11);
      }
    }
    __syncwarp();  // this warp's staging is consumed before the next block overwrites it
  }
  // per-warp row stats (quad sums) and unnormalised outputs -> smem
  l_a += __shfl_xor_sync(kFull, l_a, 1);
  l_a += __shfl_xor_sync(kFull, l_a, 2);
  l_b += __shfl_xor_sync(kFull, l_b, 1);
  l_b += __shfl_xor_sync(kFull, l_b, 2);
  __syncthreads();  // every warp is done with its K/V staging (wo reuses it)
  if (t4 == 0) {
    wm[warp][g8] = m_a;
    wl[warp][g8] = l_a;
    wm[warp][g8 + 8] = m_b;
    wl[warp][g8 + 8] = l_b;
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int d = nt * 8 + 2 * t4;
    wo[(warp * 16 + g8) * HD + d] = oacc[nt][0];
    wo[(warp * 16 + g8) * HD + d + 1] = oacc[nt][1];
    wo[(warp * 16 + g8 + 8) * HD + d] = oacc[nt][2];
    wo[(warp * 16 + g8 + 8) * HD + d + 1] = oacc[nt][3];
  }
  __syncthreads();
  if (threadIdx.x < hpg) {
    const int h = threadIdx.x;
    float M = -1e30f;
    for (int w = 0; w < NWARP; ++w) M = fmaxf(M, wm[w][h]);
    float Lsum = 0.f;
    for (int w = 0; w < NWARP; ++w) Lsum += wl[w][h] == 0.f ? 0.f : exp2f(wm[w][h] - M) * wl[w][h];
    cm_s[h] = M;
    cl_s[h] = Lsum;
  }
  __syncthreads();
  // natural-log stats for the split workspace (the combine below is shared with attention_gqa's layout)
  for (int i = threadIdx.x; i < hpg * HD; i += 128) {
    const int h = i / HD, e = i % HD;
    const float M = cm_s[h];
    float val = 0.f;
    for (int w = 0; w < NWARP; ++w)
      if (wl[w][h] != 0.f) val += exp2f(wm[w][h] - M) * wo[(w * 16 + h) * HD + e];
    const int head = g * hpg + h;
    if (nsplit == 1) {
      o[(static_cast<long long>(r) * nh + head) * HD + e] = __float2bfloat16_rn(val / cl_s[h]);
    } else {
      float* part = ws + ((static_cast<long long>(r) * nh + head) * nsplit_max + s) * (2 + HD);
      __stcg(part + 2 + e, val);
      if (e == 0) {
        __stcg(part, M * 0.6931471805599453f);  // log2 -> natural units
        __stcg(part + 1, cl_s[h]);
      }
    }
  }
  if (nsplit == 1) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt + r * nkv + g) : "memory");
    last = prev == static_cast<unsigned>(nsplit - 1);
  }
  __syncthreads();
  if (!last) return;
  // combine the splits (split order)
  float* sw_s = reinterpret_cast<float*>(KV);  // [16][64] weights
  for (int i = threadIdx.x; i < hpg * nsplit; i += 128) {
    const int h = i / nsplit, t = i % nsplit;
    sw_s[h * 64 + t] = __ldcg(ws + ((static_cast<long long>(r) * nh + g * hpg + h) * nsplit_max + t) * (2 + HD));
  }
  __syncthreads();
  if (threadIdx.x < hpg) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int t = 0; t < nsplit; ++t) M = fmaxf(M, sw_s[h * 64 + t]);
    float Lsum = 0.f;
    for (int t = 0; t < nsplit; ++t) {
      const float w = __expf(sw_s[h * 64 + t] - M);
      Lsum += w * __ldcg(ws + ((static_cast<long long>(r) * nh + g * hpg + h) * nsplit_max + t) * (2 + HD) + 1);
      sw_s[h * 64 + t] = w;
    }
    cl_s[h] = Lsum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hpg * HD; i += 128) {
    const int h = i / HD, e = i % HD;
    const float* pr = ws + (static_cast<long long>(r) * nh + g * hpg + h) * nsplit_max * (2 + HD);
    float val = 0.f;
    for (int t = 0; t < nsplit; ++t) val += sw_s[h * 64 + t] * __ldcg(pr + t * (2 + HD) + 2 + e);
    o[(static_cast<long long>(r) * nh + g * hpg + h) * HD + e] = __float2bfloat16_rn(val / cl_s[h]);
  }
  if (threadIdx.x == 0) cnt[r * nkv + g] = 0;
}

// Element index of (key, dim) in a staged key block: plain [key][HD], or (HD
// 64, TMA SWIZZLE_128B) the 16-byte chunk XOR-ed with key % 8.
__device__ __forceinline__ std::uint32_t tcpack(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&v);
}

template <int HD>
__device__ __forceinline__ long long kv_smem_index_t(int key, int d, int swz) {
  return swz ? static_cast<long long>(key) * HD + ((((d >> 3) ^ (key & 7)) << 3) | (d & 7))
             : static_cast<long long>(key) * HD + d;
}
#define kv_smem_index(key, d, swz) kv_smem_index_t<HD>((key), (d), (swz))

// ---------------------------------------------------------------------------
// Decode-tick QKV + attention in one kernel for small agents (every row is
// the only row of its agent: pure decode).  CTA = (row, kv head): its
// (hpg + 2) * hd rows of Wqkv (the group's q heads, k, v -- three contiguous
// slabs) stream into smem by bulk copy *before* the PDL wait (weights never
// depend on the previous kernel), then the row is RMS-normalised from the
// residual, the CTA computes its q/k/v columns (warp = 32 columns, lanes split
// K, one transpose-reduce), applies RoPE, appends k/v at the row's position
// and runs the group's attention (warps split the keys, online softmax,
// smem combine).  Replaces two launches and the q round trip through HBM.
constexpr int kQkvOprojMaxD = 1024;
template <int HD, int HPG>
__global__ void __launch_bounds__(256, 1)
qkv_attention_kernel(float* __restrict__ X, const float* __restrict__ g_norm, float eps, int D,
                     const bf16* __restrict__ wqkv, const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                     const float2* __restrict__ rope, int nh, int nkv, bf16* __restrict__ kpool,
                     bf16* __restrict__ vpool, long long kv_stride, long long layer_off, int max_ctx,
                     bf16* __restrict__ o, const bf16* __restrict__ emb, const int* __restrict__ out_tok,
                     int kv_cap, const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                     int tma_kv, const bf16* __restrict__ wo_blk) {
  constexpr int NW = 8, E = HD / 32, half = HD / 2;  // HPG >= q heads per kv head
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ float qs[HPG][HD];
  __shared__ float wm[NW][HPG], wl[NW][HPG];
  __shared__ float wo[NW][HPG][HD];
  __shared__ float cm_s[HPG], cl_s[HPG];
  __shared__ float red[NW];
  __shared__ __align__(8) unsigned long long wbar, obar;
  __shared__ float recv_s[kQkvOprojMaxD];  // fused o-projection: slices pushed by the cluster
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x, g = blockIdx.y;
  const int hpg = nh / nkv, ncol = (hpg + 2) * HD;
  bf16* W = reinterpret_cast<bf16*>(dsm);                          // [ncol][D]
  bf16* xn = reinterpret_cast<bf16*>(dsm + static_cast<long long>(ncol) * D * 2);  // [D]
  // keys of earlier ticks staged in smem (never produced by the previous kernel);
  // tma_kv (HD 64): 64-key TMA boxes, 128B-swizzled, 1024-aligned, for ldmatrix
  const std::uintptr_t kv_raw = reinterpret_cast<std::uintptr_t>(dsm) + static_cast<std::uintptr_t>(ncol) * D * 2 + D * 6;
  bf16* Ks = reinterpret_cast<bf16*>(tma_kv ? (kv_raw + 1023) & ~std::uintptr_t(1023) : kv_raw);  // [kv_cap][HD]
  bf16* Vs = Ks + static_cast<long long>(kv_cap) * HD;
  if (r >= __ldg(meta)) return;  // tick metadata: not produced by the previous kernel
  const RowDesc rd = rows[r];
  const int n = rd.pos + 1;
  const int ks = min(n - 1, kv_cap);  // staged earlier keys
  // keys read from smem (the own key lands there too when it fits); with the
  // swizzled TMA stage the whole context must fit (else every key from HBM)
  const bool mma_att = tma_kv && n <= kv_cap;
  const int nsm = tma_kv ? (mma_att ? n : 0) : min(n, kv_cap);
  const int kboxes = mma_att ? (ks + 63) / 64 : 0;
  const bf16* K = kpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  const bf16* V = vpool + rd.kv * kv_stride + layer_off + static_cast<long long>(g) * max_ctx * HD;
  const std::uint32_t bar = static_cast<std::uint32_t>(__cvta_generic_to_shared(&wbar));
  const unsigned stag = (2u << 16) | (emb ? 1u : 0u);
  __shared__ unsigned long long cst[kChainPhases];
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  const std::uint32_t obar_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(&obar));
  // fused o-projection: announce this CTA as started (DSMEM pushes into a
  // cluster peer wait for this before the first remote store)
  if (wo_blk) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(obar_u));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned qb = hpg * HD * D * 2, kb = HD * D * 2;
    const unsigned kvb = tma_kv ? static_cast<unsigned>(kboxes) * 64 * HD * 2 : static_cast<unsigned>(ks) * HD * 2;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(qb + 2 * kb + 2 * kvb));
    const bf16* srcs[3] = {wqkv + static_cast<long long>(g * hpg * HD) * D,
                           wqkv + static_cast<long long>((nh + g) * HD) * D,
                           wqkv + static_cast<long long>((nh + nkv + g) * HD) * D};
    const unsigned bytes[3] = {qb, kb, kb};
    unsigned off = 0;
    for (int i = 0; i < 3; ++i) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<std::uint32_t>(__cvta_generic_to_shared(dsm + off))),
          "l"(srcs[i]), "r"(bytes[i]), "r"(bar)
          : "memory");
      off += bytes[i];
    }
    if (tma_kv && kvb) {
      const int row0 = static_cast<int>((K - kpool) / HD);  // the pool as [rows][HD]
      for (int b = 0; b < kboxes; ++b) {
        tc::tma_load_2d(Ks + b * 64 * HD, &kmap, reinterpret_cast<std::uint64_t*>(&wbar), 0, row0 + b * 64);
        tc::tma_load_2d(Vs + b * 64 * HD, &vmap, reinterpret_cast<std::uint64_t*>(&wbar), 0, row0 + b * 64);
      }
    } else if (kvb) {
      const bf16* kv_src[2] = {K, V};
      bf16* kv_dst[2] = {Ks, Vs};
      for (int i = 0; i < 2; ++i)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                static_cast<std::uint32_t>(__cvta_generic_to_shared(kv_dst[i]))),
            "l"(kv_src[i]), "r"(kvb), "r"(bar)
            : "memory");
    }
  }
  for (int j = ks + threadIdx.x; j < n - 1 && j < ks + 2 * NW * 32; j += NW * 32) {  // unstaged earlier keys
    asm volatile("prefetch.global.L2 [%0];" ::"l"(K + static_cast<long long>(j) * HD));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(V + static_cast<long long>(j) * HD));
  }
  // RoPE factors of this warp's first column group (the position is tick metadata)
  float2 cs0 = make_float2(0.f, 0.f);
  if (warp < ncol / 32 && warp * 32 + lane < (hpg + 1) * HD)
    cs0 = __ldg(rope + static_cast<long long>(rd.pos) * half + ((warp * 32 + lane) % HD) / 2);
  MOA_PDL_ENTRY();
  if (threadIdx.x == 0) chain_mark(cst, 1);
  // layer 0 (emb != nullptr): the residual row is the token's embedding --
  // gathered here (the embed kernel is folded in) and written once for the
  // later kernels by the kv-head-0 CTA
  float* x = X + static_cast<long long>(r) * D;
  if (emb) {
    int tok = rd.tok;
    if (tok < 0) tok = out_tok[-1 - tok];
    const bf16* e = emb + static_cast<long long>(tok) * D;
    float* xs = reinterpret_cast<float*>(dsm + static_cast<long long>(ncol) * D * 2 + D * 2);  // [D] fp32 row
    for (int c = threadIdx.x; c < D; c += 256) {
      const float v = __bfloat162float(e[c]);
      xs[c] = v;
      if (g == 0 && !wo_blk) x[c] = v;  // fused o-projection: the owners write the final rows
    }
    __syncthreads();
    x = xs;
  }
  float ss = 0.f;
  for (int c = threadIdx.x * 4; c < D; c += 256 * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + c);
    ss = fmaf(v.x, v.x, ss);
    ss = fmaf(v.y, v.y, ss);
    ss = fmaf(v.z, v.z, ss);
    ss = fmaf(v.w, v.w, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < NW; ++w) tot += red[w];
  const float inv = 1.0f / sqrtf(tot / static_cast<float>(D) + eps);
  for (int c = threadIdx.x; c < D; c += 256) xn[c] = __float2bfloat16_rn(x[c]);  // operand bf16(x); inv scales q/k/v
  // weights landed
  {
    std::uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok)
                   : "r"(bar)
                   : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) chain_mark(cst, 3);
  // q/k/v columns: warp w takes column groups of 32 (lanes split K)
  for (int grp = warp; grp < ncol / 32; grp += NW) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    for (int k = lane * 8; k < D; k += 256) {
      float xf[8];
      unpack8(*reinterpret_cast<const uint4*>(xn + k), xf);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = dot8(xf, *reinterpret_cast<const uint4*>(W + static_cast<long long>(grp * 32 + j) * D + k), acc[j]);
    }
    const float v = transpose_reduce32(acc, lane) * inv;
    const float partner = __shfl_xor_sync(kFull, v, 1);
    const int c = grp * 32 + lane;  // column within the CTA's slab
    if (c < (hpg + 1) * HD) {       // q or k: rotate the (even, odd) pair
      const int e = (c % HD) / 2;
      const float2 cs = grp == warp ? cs0 : rope[static_cast<long long>(rd.pos) * half + e];
      const float y = (lane & 1) ? __fadd_rn(__fmul_rn(v, cs.x), __fmul_rn(partner, cs.y))
                                 : __fsub_rn(__fmul_rn(v, cs.x), __fmul_rn(partner, cs.y));
      const int d = e + ((lane & 1) ? half : 0);  // natural dim
      const bf16 yb = __float2bfloat16_rn(y);
      if (c < hpg * HD) {
        qs[c / HD][d] = __bfloat162float(yb);
      } else {
        const_cast<bf16*>(K)[static_cast<long long>(rd.pos) * HD + d] = yb;
        if (rd.pos < kv_cap) Ks[kv_smem_index(rd.pos, d, tma_kv)] = yb;
      }
    } else {
      const bf16 vb = __float2bfloat16_rn(v);
      const_cast<bf16*>(V)[static_cast<long long>(rd.pos) * HD + (c - (hpg + 1) * HD)] = vb;
      if (rd.pos < kv_cap) Vs[kv_smem_index(rd.pos, c - (hpg + 1) * HD, tma_kv)] = vb;
    }
  }
  __threadfence_block();
  // the weight slab's generic-proxy reads are ordered before the Wo bulk copy (async proxy) refills it
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) chain_mark(cst, 4);
  // fused o-projection: this group's Wo block [D][hpg*HD] into the (now free)
  // weight slab, past the 4 KB the tensor-core attention uses for its Q tile
  const int obytes = D * hpg * HD * 2;
  if (wo_blk && threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(obar_u), "r"(obytes));
    for (int off = 0; off < obytes; off += 32768) {
      const int nbytes = obytes - off < 32768 ? obytes - off : 32768;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              static_cast<std::uint32_t>(__cvta_generic_to_shared(dsm + 4096 + off))),
          "l"(reinterpret_cast<const char*>(wo_blk + static_cast<long long>(g) * D * hpg * HD) + off), "r"(nbytes),
          "r"(obar_u)
          : "memory");
    }
  }
  // attention over keys 0..pos (this row's own key included, just appended)
  if constexpr (HD == 64) {
    if (mma_att) {
      // tensor-core attention: the group's q heads are the M rows of
      // m16n8k16 tiles (Q tile in the now-free weight slab), warp w takes the
      // staged 64-key blocks w, w + 8, ... (TMA-swizzled K / V, ldmatrix)
      unsigned char* Qt = dsm;
      // keys past the own one in the last 64-key box hold whatever the pool
      // held (possibly NaN bit patterns): zero them so 0 * V stays 0
      for (int i = threadIdx.x; i < (((n + 63) & ~63) - n) * (HD / 8); i += NW * 32) {
        const int key = n + i / (HD / 8), ch = i % (HD / 8);
        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(Ks) + key * 128 + (ch << 4)) = make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(Vs) + key * 128 + (ch << 4)) = make_uint4(0, 0, 0, 0);
      }
      for (int i = threadIdx.x; i < 16 * (HD / 8); i += NW * 32) {
        const int hr = i / (HD / 8), ch = i % (HD / 8);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (hr < hpg) {
          const float* qf = &qs[hr < HPG ? hr : 0][ch * 8];
          v = make_uint4(tcpack(qf[0], qf[1]), tcpack(qf[2], qf[3]), tcpack(qf[4], qf[5]), tcpack(qf[6], qf[7]));
        }
        *reinterpret_cast<uint4*>(Qt + hr * 128 + ((ch ^ (hr & 7)) << 4)) = v;
      }
      __syncthreads();
      const std::uint32_t qt_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Qt));
      const std::uint32_t ks_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Ks));
      const std::uint32_t vs_u = static_cast<std::uint32_t>(__cvta_generic_to_shared(Vs));
      const int g8 = lane >> 2, t4 = lane & 3;
      std::uint32_t qa[4][4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int hr = lane & 15, ch = kk * 2 + (lane >> 4);
        ldsm_x4(qt_u + hr * 128 + ((ch ^ (hr & 7)) << 4), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
      }
      const float sl2 = rsqrtf(64.f) * 1.4426950408889634f;
      float m_a = -1e30f, l_a = 0.f;
      float oacc[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) oacc[nt][0] = oacc[nt][1] = oacc[nt][2] = oacc[nt][3] = 0.f;
      for (int b0k = warp * 64; b0k < n; b0k += NW * 64) {
        float sacc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
            const int krow = b0k + jp * 16 + (lane & 7) + ((lane >> 4) << 3);
            const int ch = kk * 2 + ((lane >> 3) & 1);
            std::uint32_t b00, b01, b10, b11;
            ldsm_x4(ks_u + krow * 128 + ((ch ^ (krow & 7)) << 4), b00, b01, b10, b11);
            mma_bf16(sacc[2 * jp], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b00, b01);
            mma_bf16(sacc[2 * jp + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b10, b11);
          }
        }
        float mx = -1e30f;  // rows g8 (< 8) carry the heads; rows g8 + 8 are padding
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int kq = b0k + 8 * j + 2 * t4;
          sacc[j][0] = kq < n ? sacc[j][0] * sl2 : -1e30f;
          sacc[j][1] = kq + 1 < n ? sacc[j][1] * sl2 : -1e30f;
          sacc[j][2] = sacc[j][3] = -1e30f;
          mx = fmaxf(mx, fmaxf(sacc[j][0], sacc[j][1]));
        }
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, 2));
        const float mn = fmaxf(m_a, mx), ca = exp2f(m_a - mn);
        m_a = mn;
        float ps = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          sacc[j][0] = sacc[j][0] <= -1e29f ? 0.f : exp2f(sacc[j][0] - mn);
          sacc[j][1] = sacc[j][1] <= -1e29f ? 0.f : exp2f(sacc[j][1] - mn);
          sacc[j][2] = sacc[j][3] = 0.f;
          ps += sacc[j][0] + sacc[j][1];
        }
        l_a = l_a * ca + ps;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          oacc[nt][0] *= ca;
          oacc[nt][1] *= ca;
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const std::uint32_t pa0 = tcpack(sacc[2 * kk][0], sacc[2 * kk][1]);
          const std::uint32_t pa2 = tcpack(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
#pragma unroll
          for (int np = 0; np < 4; ++np) {
            const int vrow = b0k + kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
            const int ch = np * 2 + (lane >> 4);
            std::uint32_t v00, v01, v10, v11;
            ldsm_x4_t(vs_u + vrow * 128 + ((ch ^ (vrow & 7)) << 4), v00, v01, v10, v11);
            mma_bf16(oacc[2 * np], pa0, 0u, pa2, 0u, v00, v01);
            mma_bf16(oacc[2 * np + 1], pa0, 0u, pa2, 0u, v10, v11);
          }
        }
      }
      l_a += __shfl_xor_sync(kFull, l_a, 1);
      l_a += __shfl_xor_sync(kFull, l_a, 2);
      if (g8 < hpg && g8 < HPG) {
        if (t4 == 0) {
          wm[warp][g8] = l_a == 0.f ? -INFINITY : m_a * 0.6931471805599453f;  // log2 -> natural units
          wl[warp][g8] = l_a;
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          wo[warp][g8][nt * 8 + 2 * t4] = oacc[nt][0];
          wo[warp][g8][nt * 8 + 2 * t4 + 1] = oacc[nt][1];
        }
      }
    }
  }
  if (!mma_att) {
  constexpr int TPK = HD / 64, KC = 32 / TPK;
  const int key = lane / TPK, part = lane % TPK;
  using VT = typename std::conditional<E == 2, unsigned, uint2>::type;
  const float scale = rsqrtf(static_cast<float>(HD));
  float m[HPG], l[HPG], acc[HPG][E];
#pragma unroll
  for (int h = 0; h < HPG; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[h][e] = 0.f;
  }
  for (int j0 = warp * KC; j0 < n; j0 += NW * KC) {
    const int j = j0 + key;
    // 16-byte chunk v of a key row is read as chunk (v + lane) & 7: the lanes of
    // a quarter warp hit distinct banks when the row is in smem
    // (generic loads: staged keys from smem, the rest from L2/HBM -- written by
    // earlier kernels or, for the own key, by this CTA before the barrier)
    uint4 kk[8];
    const uint4* krow = reinterpret_cast<const uint4*>((j < nsm ? Ks : K) + static_cast<long long>(j) * HD + part * 64);
#pragma unroll
    for (int v = 0; v < 8; ++v) kk[v] = j < n ? krow[(v + lane) & 7] : make_uint4(0, 0, 0, 0);
    VT vv[KC];
#pragma unroll
    for (int jj = 0; jj < KC; ++jj) {
      const int jv = j0 + jj;
      const VT* vrow = reinterpret_cast<const VT*>((jv < nsm ? Vs : V) + static_cast<long long>(jv) * HD + lane * E);
      vv[jj] = jv < n ? *vrow : VT{};
    }
#pragma unroll
    for (int h = 0; h < HPG; ++h) {
      if (h >= hpg) break;
      float dv[8];  // one partial per 16-byte chunk: 8 short FMA chains instead of one of 64
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        float f[8];
        unpack8(kk[v], f);
        const float* qv = &qs[h][part * 64 + ((v + lane) & 7) * 8];
        dv[v] = 0.f;
#pragma unroll
        for (int t = 0; t < 8; ++t) dv[v] = fmaf(qv[t], f[t], dv[v]);
      }
      float d = ((dv[0] + dv[1]) + (dv[2] + dv[3])) + ((dv[4] + dv[5]) + (dv[6] + dv[7]));
      if constexpr (TPK == 2) d += __shfl_xor_sync(kFull, d, 1);
      const float sc = j < n ? d * scale : -INFINITY;
      float cmax = sc;
#pragma unroll
      for (int off = 16; off; off >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(kFull, cmax, off));
      const float mn = fmaxf(m[h], cmax);
      const float resc = m[h] == -INFINITY ? 0.f : __expf(m[h] - mn);
      const float p = j < n ? __expf(sc - mn) : 0.f;
      l[h] = l[h] * resc + warp_sum(part == 0 ? p : 0.f);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[h][e] *= resc;
#pragma unroll
      for (int jj = 0; jj < KC; ++jj) {
        const float pj = __shfl_sync(kFull, p, jj * TPK);
        if constexpr (E == 2) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj]));
          acc[h][0] = fmaf(pj, f.x, acc[h][0]);
          acc[h][1] = fmaf(pj, f.y, acc[h][1]);
        } else {
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].x));
          const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].y));
          acc[h][0] = fmaf(pj, f0.x, acc[h][0]);
          acc[h][1] = fmaf(pj, f0.y, acc[h][1]);
          acc[h][2] = fmaf(pj, f1.x, acc[h][2]);
          acc[h][3] = fmaf(pj, f1.y, acc[h][3]);
        }
      }
      m[h] = mn;
    }
  }
#pragma unroll
  for (int h = 0; h < HPG; ++h) {
    if (h >= hpg) break;
    if (lane == 0) {
      wm[warp][h] = m[h];
      wl[warp][h] = l[h];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) wo[warp][h][lane * E + e] = acc[h][e];
  }
  }  // !mma_att
  __syncthreads();
  if (threadIdx.x == 0) chain_mark(cst, 5);
  if (threadIdx.x < hpg) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int w = 0; w < NW; ++w) M = fmaxf(M, wm[w][h]);
    float Ls = 0.f;
    for (int w = 0; w < NW; ++w) Ls += wm[w][h] == -INFINITY ? 0.f : __expf(wm[w][h] - M) * wl[w][h];
    cm_s[h] = M;
    cl_s[h] = Ls;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hpg * HD; i += NW * 32) {
    const int h = i / HD, e = i % HD;
    const float M = cm_s[h];
    float val = 0.f;
    for (int w = 0; w < NW; ++w)
      if (wm[w][h] != -INFINITY) val += __expf(wm[w][h] - M) * wo[w][h][e];
    const bf16 ob = __float2bfloat16_rn(val / cl_s[h]);
    if (wo_blk)
      qs[h][e] = __bfloat162float(ob);  // the group's attention rows stay on chip
    else
      o[(static_cast<long long>(r) * nh + g * hpg + h) * HD + e] = ob;
  }
  if (wo_blk) {
    // x[row] += o . Wo^T over the cluster of this row's kv-head CTAs: CTA g
    // forms its heads' contribution to every output column, pushes slice q of
    // it into CTA q's smem (DSMEM), and CTA q adds the slices in rank order
    // to the residual and writes its D / nkv columns
    // (the receive slices are a dedicated static buffer: pushes need no
    // barrier before them, only the one that publishes them)
    const int S = D / nkv;
    float* recv = recv_s;  // [nkv][S]
    __syncthreads();
    {
      std::uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok)
                     : "r"(obar_u)
                     : "memory");
    }
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // every peer has started
    const int K8 = hpg * HD / 8;  // 16-byte chunks per Wo row
    const bf16* wob = reinterpret_cast<const bf16*>(dsm + 4096);
    for (int n = threadIdx.x; n < D; n += NW * 32) {
      const uint4* wr = reinterpret_cast<const uint4*>(wob + static_cast<long long>(n) * hpg * HD);
      float acc = 0.f;
      for (int c = 0; c < K8; ++c) {
        const int cr = (c + n) % K8;  // rotated: the rows of a quarter warp hit distinct banks
        float w8[8];
        unpack8(wr[cr], w8);
        const int h = (cr * 8) / HD, d0 = (cr * 8) % HD;
#pragma unroll
        for (int t = 0; t < 8; ++t) acc = fmaf(qs[h][d0 + t], w8[t], acc);
      }
      const int q = n / S, i = n % S;
      std::uint32_t dst;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                   : "=r"(dst)
                   : "r"(static_cast<std::uint32_t>(__cvta_generic_to_shared(recv + g * S + i))), "r"(q));
      asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst), "f"(acc) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int i = threadIdx.x; i < S; i += NW * 32) {
      float v = x[g * S + i];
      for (int src = 0; src < nkv; ++src) v += recv[src * S + i];
      X[static_cast<long long>(r) * D + g * S + i] = v;
    }
  }
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, stag);
  }
}

// LM head: block b owns a contiguous vocab slice; warps take 4 columns x 8
// rows at a time; rows are normalised on the fly.  The last CTA merges all
// slices per row in slice order and writes token / logprob / entropy.
constexpr int kLmBlocksPerSm = 4;

__global__ void __launch_bounds__(kWarps * 32)
lm_head_kernel(const float* __restrict__ X, const int* __restrict__ sel, const int* __restrict__ meta,
               const float* __restrict__ g,
               float eps, const bf16* __restrict__ W, int V, int d, LmStat* __restrict__ part,
               int* __restrict__ cnt, const int* __restrict__ out_idx, int* __restrict__ out_tok,
               float* __restrict__ out_lp, float* __restrict__ out_ent, float* __restrict__ logits) {
  MOA_PDL_ENTRY();
  __shared__ float inv_s[kLmMaxRows];
  __shared__ LmStat sm[kWarps][kRB];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  const int per = (V + nb - 1) / nb;
  const int c0 = blockIdx.x * per, c1 = min(V, c0 + per);
  const int Rl = __ldg(meta + 1);
  if (Rl <= 0) return;
  for (int r = warp; r < Rl; r += kWarps) {
    const float inv = row_inv_rms(X + static_cast<long long>(sel[r]) * d, d, eps, lane);
    if (lane == 0) inv_s[r] = inv;
  }
  __syncthreads();
  GemvArgs ga;
  ga.X = X;
  ga.K = d;
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
            float f[8];
            load_a<true>(ga, sel[r0 + r], k, f);
#pragma unroll
            for (int c = 0; c < kCPW; ++c) acc[c * kRB + r] = dot8(f, w[c], acc[c * kRB + r]);
          }
        }
      }
      const int c = lane / kRB, r = lane % kRB;
      const float v = transpose_reduce32(acc, lane) * (r < rows ? inv_s[r0 + r] : 0.f);
      if (r < rows && cb + c < c1) {
        if (logits) logits[static_cast<long long>(r0 + r) * V + cb + c] = v;
        st = stat_merge(st, LmStat{v, 1.f, 0.f, cb + c});
      }
    }
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) {
      const LmStat o = shfl_stat(st, off);
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
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(cnt, 1) == nb - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int r = warp; r < Rl; r += kWarps) {
    LmStat st{-INFINITY, 0.f, 0.f, INT_MAX};
    const float4* pr = reinterpret_cast<const float4*>(part + static_cast<long long>(r) * nb);
    // issue the lane's partial loads in batches of 8 before merging them
    for (int b0 = lane; b0 < nb; b0 += 32 * 8) {
      float4 raw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + 32 * u;
        raw[u] = b < nb ? __ldcg(pr + b) : make_float4(-INFINITY, 0.f, 0.f, __int_as_float(INT_MAX));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) st = stat_merge(st, LmStat{raw[u].x, raw[u].y, raw[u].z, __float_as_int(raw[u].w)});
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const LmStat o = shfl_stat(st, off);
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
  if (threadIdx.x == 0) *cnt = 0;
}

// chain-overhead probe: waits for its predecessor, releases its dependents,
// touches one int
__global__ void noop_kernel(int* p) {
  MOA_PDL_ENTRY();
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  return static_cast<int>(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

template <bool NORM>
void gemv_launch(const GemvArgs& a, cudaStream_t st) {
  // k-parts per CTA: as many as K allows (each part a multiple of 256)
  int kp = 8;
  while (kp > 1 && (a.K % (256 * kp))) kp >>= 1;
  const int wg = kWarps / kp;
  dim3 grid((a.N + wg * kCPW - 1) / (wg * kCPW), 1, (a.R + kRB - 1) / kRB);
  switch (wg) {
    case 1: launch_pdl(gemv_kernel<1, NORM>, grid, dim3(kWarps * 32), st, a); break;
    case 2: launch_pdl(gemv_kernel<2, NORM>, grid, dim3(kWarps * 32), st, a); break;
    case 4: launch_pdl(gemv_kernel<4, NORM>, grid, dim3(kWarps * 32), st, a); break;
    default: launch_pdl(gemv_kernel<8, NORM>, grid, dim3(kWarps * 32), st, a); break;
  }
}

}  // namespace

void init_uniform_rows(bf16* dst, long long rows, long long cols, std::uint64_t base, float scale, int map, int hd,
                       cudaStream_t st) {
  init_uniform_rows_kernel<<<grid_for(rows * cols, 256), 256, 0, st>>>(dst, rows, cols, base, scale, map, hd);
}

void noop_chain_link(int* p, int ctas, cudaStream_t st) { launch_pdl(noop_kernel, dim3(ctas), dim3(128), st, p); }

void fill_f32(float* dst, long long n, float v, cudaStream_t st) {
  fill_f32_kernel<<<grid_for(n, 256), 256, 0, st>>>(dst, n, v);
}

void embed(const RowDesc* rows, int R_cap, const int* meta, const int* out_tok, const bf16* emb, int d, float* x,
           cudaStream_t st, float* ssq, bf16* xb) {
  if (R_cap > 0) launch_pdl(embed_kernel, dim3(R_cap), dim3(128), st, rows, meta, out_tok, emb, d, x, ssq, xb);
}

void gemv(const GemvArgs& a, cudaStream_t st) {
  if (a.R <= 0) return;
  if (gemv_stream_supported(a)) {
    gemv_stream(a, st);
    return;
  }
  if (a.X)
    gemv_launch<true>(a, st);
  else
    gemv_launch<false>(a, st);
}

long long attention_ws_floats(int R, int nh, int hd, int max_ctx) {
  const int ns = (max_ctx + kKvSplit - 1) / kKvSplit;
  return static_cast<long long>(R) * nh * ns * (2 + hd);
}

void attention(const bf16* q, const RowDesc* rows, int R_cap, int nsplit_cap, const int* meta, int nh, int nkv, int hd,
               const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off, int max_ctx, bf16* o,
               float* ws, int* cnt, cudaStream_t st, bool skip_runs) {
  if (R_cap <= 0) return;
  const int nsplit_max = (max_ctx + kKvSplit - 1) / kKvSplit;
  const int split_keys = kv_split(hd);
  // q heads per CTA: MOA_ATTN_HPC (1, 2 or 4); default: the whole GQA group
  // (measured: one CTA per q head re-reads K/V per head -- 1.5x slower on
  // 2k-token 8B contexts, 6% slower on 1B decode)
  static const int hpc_env = [] {
    const char* e = std::getenv("MOA_ATTN_HPC");
    return e ? std::atoi(e) : 4;
  }();
  const int hpg = nh / nkv;
  static const bool mma = [] {  // MOA_DECODE_MMA=0: the SIMT kernel
    const char* e = std::getenv("MOA_DECODE_MMA");
    return !(e && e[0] == '0');
  }();
  if (mma && hpg <= 16 && nsplit_max <= 64) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(R_cap, nkv, nsplit_cap);
    cfg.blockDim = dim3(128);
    const int smem = 16 * hd * 2 + 4 * 2 * kPfKeys * hd * 2;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    auto gm = [&](auto kern) {
      static std::set<const void*> attr;
      if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        uniform_carveout(reinterpret_cast<const void*>(kern));
      }
      cudaLaunchKernelEx(&cfg, kern, q, rows, meta, nh, nkv, kpool, vpool, kv_stride, layer_off, max_ctx, o, ws, cnt,
                         nsplit_max, split_keys, skip_runs ? 1 : 0);
    };
    if (hd == 64)
      gm(attention_decode_mma_kernel<64>);
    else
      gm(attention_decode_mma_kernel<128>);
    return;
  }
  int hpc = hpc_env == 2 || hpc_env == 4 ? hpc_env : 1;
  while (hpg % hpc) hpc >>= 1;
  dim3 grid(R_cap, nh / hpc, nsplit_cap);
  auto go = [&](auto kern) {
    launch_pdl(kern, grid, dim3(256), st, q, rows, meta, nh, nkv, kpool, vpool, kv_stride, layer_off, max_ctx, o, ws,
               cnt, nsplit_max, split_keys, skip_runs ? 1 : 0);
  };
  if (hd == 64) {
    if (hpc == 1) go(attention_gqa_kernel<64, 1>);
    else if (hpc == 2) go(attention_gqa_kernel<64, 2>);
    else go(attention_gqa_kernel<64, 4>);
  } else if (hd == 128) {
    if (hpc == 1) go(attention_gqa_kernel<128, 1>);
    else if (hpc == 2) go(attention_gqa_kernel<128, 2>);
    else go(attention_gqa_kernel<128, 4>);
  } else {
    printf("attention: unsupported head_dim %d\n", hd);
  }
}

MOA_CHAIN_STAMP_SETTER(forward_chain_stamp)

void attention_prefill(const bf16* q, const RowDesc* rows, int R_cap, const int* meta, int nh, int nkv, int hd,
                       const bf16* kpool, const bf16* vpool, long long kv_stride, long long layer_off, int max_ctx,
                       bf16* o, cudaStream_t st) {
  static const bool mma = [] {  // MOA_PREFILL_MMA=0: the SIMT kernel
    const char* e = std::getenv("MOA_PREFILL_MMA");
    return !(e && e[0] == '0');
  }();
  const int smem = mma ? (kPfRows + 2 * kPfKeys) * hd * 2
                       : (hd * (kPfKeys + 1) + kPfKeys * hd + 8 * 8 * hd + 8 * kPfKeys * 8) * 4;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((R_cap + kPfRows - 1) / kPfRows, nh);
  cfg.blockDim = dim3(mma ? 128 : 256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  auto go = [&](auto kern) {
    static std::set<const void*> attr;
    if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      uniform_carveout(reinterpret_cast<const void*>(kern));
    }
    cudaLaunchKernelEx(&cfg, kern, q, rows, meta, nh, nkv, kpool, vpool, kv_stride, layer_off, max_ctx, o);
  };
  if (mma) {
    if (hd == 64)
      go(attention_prefill_mma_kernel<64>);
    else
      go(attention_prefill_mma_kernel<128>);
  } else if (hd == 64) {
    go(attention_prefill_kernel<64>);
  } else {
    go(attention_prefill_kernel<128>);
  }
}

int qkv_attention_smem(int D, int nh, int nkv, int hd) { return ((nh / nkv) + 2) * hd * D * 2 + D * 2 + D * 4 + 128; }
// earlier keys one CTA stages in smem next to its weight slab (<= 200 KB of
// dynamic smem: the kernel's static arrays take up to ~19 KB of the 227)
static int qkv_attention_kv_cap(int D, int nh, int nkv, int hd, int max_ctx) {
  static const int limit = [] {  // MOA_QKV_KV_STAGE=n caps the staged keys (0: none; tests)
    const char* e = std::getenv("MOA_QKV_KV_STAGE");
    return e ? std::atoi(e) : 1 << 30;
  }();
  int c = (200 * 1024 - qkv_attention_smem(D, nh, nkv, hd)) / (hd * 4);
  c = std::min({c, max_ctx, limit});
  return c < 0 ? 0 : c;
}

bool qkv_attention_supported(int D, int nh, int nkv, int hd) {
  return (hd == 64 || hd == 128) && nh % nkv == 0 && nh / nkv <= 4 && D % 256 == 0 &&
         (((nh / nkv) + 2) * hd) % 32 == 0 && qkv_attention_smem(D, nh, nkv, hd) <= 160 * 1024;
}

bool qkv_oproj_supported(int D, int nh, int nkv, int hd) {
  // the Wo block must fit the freed weight slab, the pushed slices the receive buffer
  return qkv_attention_supported(D, nh, nkv, hd) && D % nkv == 0 && nkv <= 8 && D <= kQkvOprojMaxD &&
         4096 + D * (nh / nkv) * hd * 2 <= ((nh / nkv) + 2) * hd * D * 2;
}

void qkv_attention(float* X, const float* g, float eps, int D, const bf16* wqkv, const RowDesc* rows, int R_cap,
                   const int* meta, const float2* rope, int nh, int nkv, int hd, bf16* kpool, bf16* vpool,
                   long long kv_stride, long long layer_off, int max_ctx, bf16* o, cudaStream_t st, const bf16* emb,
                   const int* out_tok, const TmaMap* kmap, const TmaMap* vmap, const bf16* wo_blk) {
  static const bool mma_env = [] {  // MOA_QKV_MMA=0: SIMT attention phase
    const char* e = std::getenv("MOA_QKV_MMA");
    return !(e && e[0] == '0');
  }();
  const int tma_kv = (mma_env && hd == 64 && kmap && vmap) ? 1 : 0;
  int kv_cap = qkv_attention_kv_cap(D, nh, nkv, hd, max_ctx);
  if (tma_kv) kv_cap = (kv_cap - 1024 / (hd * 4)) / 64 * 64;  // whole 64-key boxes after the 1 KB alignment pad
  const int smem = qkv_attention_smem(D, nh, nkv, hd) + kv_cap * hd * 4 + (tma_kv ? 1024 : 0);
  if (wo_blk && !qkv_oproj_supported(D, nh, nkv, hd)) {
    // the caller dropped its o-projection launch: silently skipping it here would lose the projection
    std::fprintf(stderr, "qkv_attention: fused o-projection requested for an unsupported shape\n");
    std::abort();
  }
  static const CUtensorMap no_map{};
  const CUtensorMap& km = tma_kv ? *reinterpret_cast<const CUtensorMap*>(kmap) : no_map;
  const CUtensorMap& vm = tma_kv ? *reinterpret_cast<const CUtensorMap*>(vmap) : no_map;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(R_cap, nkv);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (wo_blk) {  // a row's kv-head CTAs form one cluster (the fused o-projection exchanges over DSMEM)
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1;
    at[na].val.clusterDim.y = nkv;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const int hpg = nh / nkv;
  auto go = [&](auto kern) {
    static std::set<const void*> attr;
    if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      uniform_carveout(reinterpret_cast<const void*>(kern));
    }
    cudaLaunchKernelEx(&cfg, kern, X, g, eps, D, wqkv, rows, meta, rope, nh, nkv, kpool, vpool, kv_stride, layer_off,
                       max_ctx, o, emb, out_tok, kv_cap, km, vm, tma_kv, wo_blk);
  };
  if (hd == 64) {
    if (hpg == 1) go(qkv_attention_kernel<64, 1>);
    else if (hpg == 2) go(qkv_attention_kernel<64, 2>);
    else go(qkv_attention_kernel<64, 4>);
  } else {
    if (hpg == 1) go(qkv_attention_kernel<128, 1>);
    else if (hpg == 2) go(qkv_attention_kernel<128, 2>);
    else go(qkv_attention_kernel<128, 4>);
  }
}

int lm_head_blocks(int V) {
  int nb = 148 * kLmBlocksPerSm;
  return nb < V ? nb : V;
}

void lm_head(const float* X, const int* sel, const int* meta, const float* g, float eps, const bf16* W, int V, int d,
             LmStat* part, int* cnt, const int* out_idx, int* out_tok, float* out_lp, float* out_ent, float* logits,
             cudaStream_t st) {
  launch_pdl(lm_head_kernel, dim3(lm_head_blocks(V)), dim3(kWarps * 32), st, X, sel, meta, g, eps, W, V, d, part, cnt, out_idx, out_tok,
                                                            out_lp, out_ent, logits);
}

}  // namespace moa::k
