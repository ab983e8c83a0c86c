// Cluster-resident decode forward for small agents (the `tiny` shape: d <= 512,
// ffn <= 1024): all transformer layers of a tick of <= 16 rows in ONE launch
// of one 16-CTA thread-block cluster.
//
// Why: a `tiny` forward is ~23 short kernels whose cost is the kernel
// boundary (grid drain + memory flush + the next kernel's first global round
// trip), not bytes -- its layer weights are 8 MB.  Inside one cluster the
// boundaries become cluster barriers and the activations never leave shared
// memory:
//
//   * every CTA keeps a replica of the residual rows x [R][d] (fp32), the
//     SwiGLU rows h [R][ffn], the rotated queries q and the attention output
//     o (bf16) in its shared memory;
//   * CTA c owns a 1/16 column slab of every weight matrix; slabs stream from
//     L2/HBM with cp.async.bulk into a 2-slot ring one step ahead of use (the
//     first two before griddepcontrol.wait -- weights never depend on the
//     previous kernel);
//   * each GEMV step computes the CTA's columns for all rows (RMSNorm applied
//     on the fly from the local replica; a warp reduces 32/RP columns x RP
//     rows at once, RP = rows rounded up to 4/8/16), runs the fused epilogue
//     (RoPE + KV append, residual, SwiGLU) into a local slice, and copies the
//     slice into all 16 replicas with 16-byte st.shared::cluster stores
//     (DSMEM), then one cluster barrier;  q is kept in the weights' RoPE-pair
//     order (contiguous per CTA) and reordered per attention unit;
//   * attention: CTA c takes (row, kv head) units c, c+16, ...; its 8 warps
//     split the keys with an online softmax per head, combine in smem, and
//     broadcast the unit's output rows.
//
// The LM head (25.6 MB for `tiny`) stays a separate persistent kernel over
// every SM: this kernel writes the final rows of x to global memory and
// triggers it early (PDL).
//
// Rounding points are the oracle's (bf16 GEMM operands, fp32 accumulation and
// residual, bf16 KV); reduction orders are fixed (results do not depend on
// timing or on which rows share the tick).
#include <cstdio>
#include <type_traits>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace moa::k {

namespace {

using namespace tc;

constexpr int CS = kSmallCluster;  // CTAs per cluster
constexpr int NT = 256, NW = 8;
constexpr int RMAX = kMkRows;  // rows per tick
constexpr int kSlot = kSmallSlotBytes;

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ std::uint32_t remote(std::uint32_t local, unsigned rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}

// write one value into the same smem location of every CTA of the cluster
// Copy a [rows][bytes_per_row] slice (local smem, row stride src_stride)
// into the same place of every CTA's replica (row stride dst_stride), 16 B per
// store; all threads of the CTA participate.
__device__ __forceinline__ void bcast_slice(const unsigned char* src, int src_stride, unsigned char* dst_local,
                                            int dst_stride, int rows, int bytes_per_row) {
  const int chunks = bytes_per_row / 16, per_dest = rows * chunks;
  const std::uint32_t d0 = smem_u32(dst_local);
  for (int i = threadIdx.x; i < CS * per_dest; i += NT) {
    const unsigned q = static_cast<unsigned>(i / per_dest);
    const int rem = i % per_dest, r = rem / chunks, ch = rem % chunks;
    const uint4 v = *reinterpret_cast<const uint4*>(src + r * src_stride + ch * 16);
    const std::uint32_t a = remote(d0 + r * dst_stride + ch * 16, q);
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void unpack8(uint4 a, float (&f)[8]) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 u = __bfloat1622float2(x[i]);
    f[2 * i] = u.x;
    f[2 * i + 1] = u.y;
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// lane L ends with the sum over lanes of v[L] (31 shuffles for 32 values)
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool upper = lane & off;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = upper ? v[i] : v[i + off];
      const float keep = upper ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

struct Sm {
  unsigned char* w[2];
  float* xs;   // [RMAX][D]    residual replica
  bf16* hs;    // [RMAX][ffn]  SwiGLU replica
  bf16* qs;    // [RMAX][QD]   queries, RoPE-pair order (the weights' row order)
  bf16* os;    // [RMAX][QD]   attention output
  unsigned char* st;  // [RMAX][kStageBytes] this CTA's output slice before the broadcast
  float* qn;   // [4][hd]      one unit's queries, natural order
  float* inv;  // [RMAX]
  std::uint64_t* bar;  // [2]
  float* wm;   // [NW][4]
  float* wl;   // [NW][4]
  float* wo;   // [NW][4][hd]
  float* cm;   // [4]
  float* cl;   // [4]
};
constexpr int kStageBytes = 512;  // per-row slice: <= 128 fp32 / 256 bf16 columns

__device__ __forceinline__ Sm carve(unsigned char* raw, const SmallParams& P) {
  unsigned char* p =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(raw) + 127) & ~std::uintptr_t(127));
  const int QD = P.nh * P.hd;
  Sm s;
  s.w[0] = p;
  p += kSlot;
  s.w[1] = p;
  p += kSlot;
  s.xs = reinterpret_cast<float*>(p);
  p += RMAX * P.D * 4;
  s.hs = reinterpret_cast<bf16*>(p);
  p += RMAX * P.ffn * 2;
  s.qs = reinterpret_cast<bf16*>(p);
  p += RMAX * QD * 2;
  s.os = reinterpret_cast<bf16*>(p);
  p += RMAX * QD * 2;
  s.st = p;
  p += RMAX * kStageBytes;
  s.qn = reinterpret_cast<float*>(p);
  p += 4 * P.hd * 4;
  s.wo = reinterpret_cast<float*>(p);
  p += NW * 4 * P.hd * 4;
  s.wm = reinterpret_cast<float*>(p);
  p += NW * 4 * 4;
  s.wl = reinterpret_cast<float*>(p);
  p += NW * 4 * 4;
  s.cm = reinterpret_cast<float*>(p);
  p += 16;
  s.cl = reinterpret_cast<float*>(p);
  p += 16;
  s.inv = reinterpret_cast<float*>(p);
  p += RMAX * 4;
  s.bar = reinterpret_cast<std::uint64_t*>((reinterpret_cast<std::uintptr_t>(p) + 7) & ~std::uintptr_t(7));
  return s;
}

// The CTA's columns [0, ncols) of W (a slab in smem, [ncols][K]) for rows < R:
// warp w takes column groups w, w+8, ... of CG = 32/RP columns; lanes split K
// in 8-element chunks; one transpose-reduce per group.  Activations: NORM ->
// bf16(x * inv * g) from the x replica, else bf16 rows xb[r][K].
// epi(col, row, value, partner): lane L holds column CG*grp + L/RP, row L%RP;
// partner = the other column of the even/odd pair, same row.
template <int RP, bool NORM, class Epi>
__device__ __forceinline__ void slab_gemv(const bf16* __restrict__ W, int ncols, int K, const Sm& sm, int D,
                                          const float* __restrict__ g, const bf16* xb, int R, Epi&& epi) {
  constexpr int CG = 32 / RP;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int grp = warp; grp < ncols / CG; grp += NW) {
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    const bf16* wg = W + static_cast<long long>(grp * CG) * K;
    for (int k = lane * 8; k < K; k += 256) {
      uint4 wr[CG];
#pragma unroll
      for (int cc = 0; cc < CG; ++cc) wr[cc] = *reinterpret_cast<const uint4*>(wg + static_cast<long long>(cc) * K + k);
      float4 g0 = make_float4(1.f, 1.f, 1.f, 1.f), g1 = g0;
      if constexpr (NORM) {
        g0 = __ldg(reinterpret_cast<const float4*>(g + k));
        g1 = __ldg(reinterpret_cast<const float4*>(g + k + 4));
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) break;
        float xv[8];
        if constexpr (NORM) {
          const float4 x0 = *reinterpret_cast<const float4*>(sm.xs + r * D + k);
          const float4 x1 = *reinterpret_cast<const float4*>(sm.xs + r * D + k + 4);
          const float iv = sm.inv[r];
          xv[0] = __bfloat162float(__float2bfloat16_rn(x0.x * iv * g0.x));
          xv[1] = __bfloat162float(__float2bfloat16_rn(x0.y * iv * g0.y));
          xv[2] = __bfloat162float(__float2bfloat16_rn(x0.z * iv * g0.z));
          xv[3] = __bfloat162float(__float2bfloat16_rn(x0.w * iv * g0.w));
          xv[4] = __bfloat162float(__float2bfloat16_rn(x1.x * iv * g1.x));
          xv[5] = __bfloat162float(__float2bfloat16_rn(x1.y * iv * g1.y));
          xv[6] = __bfloat162float(__float2bfloat16_rn(x1.z * iv * g1.z));
          xv[7] = __bfloat162float(__float2bfloat16_rn(x1.w * iv * g1.w));
        } else {
          unpack8(*reinterpret_cast<const uint4*>(xb + r * K + k), xv);
        }
#pragma unroll
        for (int cc = 0; cc < CG; ++cc) {
          float f[8];
          unpack8(wr[cc], f);
#pragma unroll
          for (int t = 0; t < 8; ++t) acc[cc * RP + r] = fmaf(xv[t], f[t], acc[cc * RP + r]);
        }
      }
    }
    const float v = transpose_reduce32(acc, lane);
    const float partner = __shfl_xor_sync(0xffffffffu, v, RP);
    epi(grp * CG + lane / RP, lane % RP, v, partner);
  }
}

// row inverse RMS of the x replica: warp w handles rows w, w + 8
__device__ __forceinline__ void row_norms(const Sm& sm, int D, float eps, int R) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < R; r += NW) {
    float ss = 0.f;
    for (int k = lane * 4; k < D; k += 128) {
      const float4 v = *reinterpret_cast<const float4*>(sm.xs + r * D + k);
      ss = fmaf(v.x, v.x, ss);
      ss = fmaf(v.y, v.y, ss);
      ss = fmaf(v.z, v.z, ss);
      ss = fmaf(v.w, v.w, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) sm.inv[r] = 1.0f / sqrtf(ss / static_cast<float>(D) + eps);
  }
}

// attention units (row, kv head) c, c+16, ...: the 8 warps split the keys,
// online softmax per head of the group, combine in smem, broadcast o.
template <int HD>
__device__ void attention_step(const SmallParams& P, int layer, int R, const Sm& sm, unsigned c) {
  constexpr int TPK = HD / 64, KC = 32 / TPK, E = HD / 32, half = HD / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int key = lane / TPK, part = lane % TPK;
  const int hpg = P.nh / P.nkv, QD = P.nh * HD;
  const long long loff = P.layer_stride * layer;
  const float scale = rsqrtf(static_cast<float>(HD));
  using VT = typename std::conditional<E == 2, unsigned, uint2>::type;
  for (int u = static_cast<int>(c); u < R * P.nkv; u += CS) {
    const int r = u / P.nkv, g = u % P.nkv;
    // the group's queries, RoPE-pair order -> natural order (fp32)
    for (int i = threadIdx.x; i < hpg * HD; i += NT) {
      const int h = i / HD, d = i % HD;
      const int src = d < half ? 2 * d : 2 * (d - half) + 1;
      sm.qn[i] = __bfloat162float(sm.qs[r * QD + (g * hpg + h) * HD + src]);
    }
    __syncthreads();
    const RowDesc rd = P.rows[r];
    const int n = rd.pos + 1;
    const bf16* K = P.kpool + rd.kv * P.kv_stride + loff + static_cast<long long>(g) * P.max_ctx * HD;
    const bf16* V = P.vpool + rd.kv * P.kv_stride + loff + static_cast<long long>(g) * P.max_ctx * HD;
    float m[4], l[4], acc[4][E];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      m[h] = -INFINITY;
      l[h] = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[h][e] = 0.f;
    }
    for (int j0 = warp * KC; j0 < n; j0 += NW * KC) {
      const int j = j0 + key;
      uint4 kk[8];
#pragma unroll
      for (int v = 0; v < 8; ++v)
        kk[v] = j < n ? __ldcg(reinterpret_cast<const uint4*>(K + static_cast<long long>(j) * HD + part * 64) + v)
                      : make_uint4(0, 0, 0, 0);
      VT vv[KC];
#pragma unroll
      for (int jj = 0; jj < KC; ++jj)
        vv[jj] = j0 + jj < n ? __ldcg(reinterpret_cast<const VT*>(V + static_cast<long long>(j0 + jj) * HD + lane * E))
                             : VT{};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        if (h >= hpg) break;
        const float* qh = sm.qn + h * HD + part * 64;
        float d = 0.f;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          float f[8];
          unpack8(kk[v], f);
          const float4 q0 = *reinterpret_cast<const float4*>(qh + v * 8);
          const float4 q1 = *reinterpret_cast<const float4*>(qh + v * 8 + 4);
          d = fmaf(q0.x, f[0], d);
          d = fmaf(q0.y, f[1], d);
          d = fmaf(q0.z, f[2], d);
          d = fmaf(q0.w, f[3], d);
          d = fmaf(q1.x, f[4], d);
          d = fmaf(q1.y, f[5], d);
          d = fmaf(q1.z, f[6], d);
          d = fmaf(q1.w, f[7], d);
        }
        if constexpr (TPK == 2) d += __shfl_xor_sync(0xffffffffu, d, 1);
        const float sc = j < n ? d * scale : -INFINITY;
        float cmax = sc;
#pragma unroll
        for (int off = 16; off; off >>= 1) cmax = fmaxf(cmax, __shfl_xor_sync(0xffffffffu, cmax, off));
        const float mn = fmaxf(m[h], cmax);
        const float resc = m[h] == -INFINITY ? 0.f : __expf(m[h] - mn);
        const float p = j < n ? __expf(sc - mn) : 0.f;
        l[h] = l[h] * resc + warp_sum(part == 0 ? p : 0.f);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[h][e] *= resc;
#pragma unroll
        for (int jj = 0; jj < KC; ++jj) {
          const float pj = __shfl_sync(0xffffffffu, p, jj * TPK);
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
    for (int h = 0; h < 4; ++h) {
      if (h >= hpg) break;
      if (lane == 0) {
        sm.wm[warp * 4 + h] = m[h];
        sm.wl[warp * 4 + h] = l[h];
      }
#pragma unroll
      for (int e = 0; e < E; ++e) sm.wo[(warp * 4 + h) * HD + lane * E + e] = acc[h][e];
    }
    __syncthreads();
    if (threadIdx.x < hpg) {
      const int h = threadIdx.x;
      float M = -INFINITY;
      for (int w = 0; w < NW; ++w) M = fmaxf(M, sm.wm[w * 4 + h]);
      float Ls = 0.f;
      for (int w = 0; w < NW; ++w)
        Ls += sm.wm[w * 4 + h] == -INFINITY ? 0.f : __expf(sm.wm[w * 4 + h] - M) * sm.wl[w * 4 + h];
      sm.cm[h] = M;
      sm.cl[h] = Ls;
    }
    __syncthreads();
    bf16* stg = reinterpret_cast<bf16*>(sm.st);  // one row: the group's hpg * HD outputs
    for (int i = threadIdx.x; i < hpg * HD; i += NT) {
      const int h = i / HD, e = i % HD;
      const float M = sm.cm[h];
      float val = 0.f;
      for (int w = 0; w < NW; ++w)
        if (sm.wm[w * 4 + h] != -INFINITY) val += __expf(sm.wm[w * 4 + h] - M) * sm.wo[(w * 4 + h) * HD + e];
      stg[i] = __float2bfloat16_rn(val / sm.cl[h]);
    }
    __syncthreads();
    bcast_slice(sm.st, 0, reinterpret_cast<unsigned char*>(sm.os + r * QD + g * hpg * HD), 0, 1, hpg * HD * 2);
    __syncthreads();  // staging / wm / wo reused by the next unit
  }
}

__device__ unsigned long long* g_small_trace = nullptr;  // debug: [cta][64] clock64 stamps
__device__ __forceinline__ void sstamp(int ev) {
  if (g_small_trace && threadIdx.x == 0) g_small_trace[cluster_rank() * 64 + ev] = clock64();
}

template <int RP>
__device__ void run_layers(const SmallParams& P, const Sm& sm, unsigned c, int R) {
  const int D = P.D, QD = P.nh * P.hd, FF = P.ffn, L = P.L, hd = P.hd, half = hd / 2;
  const int qkv_cols = (P.nh + 2 * P.nkv) * hd;
  const int nq = qkv_cols / CS, no = D / CS, ng = 2 * FF / CS, nd = D / CS;
  const int nslab = 4 * L;
  auto slab_src = [&](int s, unsigned* bytes) -> const bf16* {
    const int l = s / 4, j = s % 4;
    const bf16* base = P.w0 + static_cast<long long>(l) * P.wstride;
    switch (j) {
      case 0: *bytes = nq * D * 2; return base + static_cast<long long>(c) * nq * D;
      case 1: *bytes = no * QD * 2; return base + P.off_o + static_cast<long long>(c) * no * QD;
      case 2: *bytes = ng * D * 2; return base + P.off_gu + static_cast<long long>(c) * ng * D;
      default: *bytes = nd * FF * 2; return base + P.off_d + static_cast<long long>(c) * nd * FF;
    }
  };
  float* stf = reinterpret_cast<float*>(sm.st);
  bf16* stb = reinterpret_cast<bf16*>(sm.st);
  constexpr int SF = kStageBytes / 4, SB = kStageBytes / 2;  // staging row strides (fp32 / bf16 elements)
  for (int l = 0; l < L; ++l) {
    const long long loff = P.layer_stride * l;
    for (int j = 0; j < 4; ++j) {
      const int s = 4 * l + j, slot = s & 1;
      if (j == 0 || j == 2) {
        row_norms(sm, D, P.eps, R);
        __syncthreads();
      }
      mbar_wait(&sm.bar[slot], (s >> 1) & 1);
      if (l == 1) sstamp(3 + j * 4);
      const bf16* W = reinterpret_cast<const bf16*>(sm.w[slot]);
      if (j == 0) {  // QKV + RoPE; q slice staged, K/V appended to the pool
        const int n0 = static_cast<int>(c) * nq;
        slab_gemv<RP, true>(W, nq, D, sm, D, P.g, nullptr, R, [&](int cl, int r, float v, float partner) {
          if (r >= R) return;
          const int n = n0 + cl;
          const RowDesc rd = P.rows[r];
          if (n < (P.nh + P.nkv) * hd) {
            const int head = n / hd, e = (n % hd) / 2;
            const float2 cs = P.rope[static_cast<long long>(rd.pos) * half + e];
            // even member: x0 = v, x1 = partner -> y0; odd member: x1 = v, x0 = partner -> y1
            const float y = (n & 1) ? __fadd_rn(__fmul_rn(v, cs.x), __fmul_rn(partner, cs.y))
                                    : __fsub_rn(__fmul_rn(v, cs.x), __fmul_rn(partner, cs.y));
            if (head < P.nh) {
              stb[r * SB + cl] = __float2bfloat16_rn(y);
            } else {
              bf16* dst = P.kpool + rd.kv * P.kv_stride + loff +
                          (static_cast<long long>(head - P.nh) * P.max_ctx + rd.pos) * hd;
              dst[e + ((n & 1) ? half : 0)] = __float2bfloat16_rn(y);
            }
          } else {
            const int vc = n - (P.nh + P.nkv) * hd, kh = vc / hd, e = vc % hd;
            P.vpool[rd.kv * P.kv_stride + loff + (static_cast<long long>(kh) * P.max_ctx + rd.pos) * hd + e] =
                __float2bfloat16_rn(v);
          }
        });
        __syncthreads();
        if (l == 1) sstamp(4);
        const int q_end = min(n0 + nq, QD);  // this CTA's q columns [n0, q_end)
        if (q_end > n0)
          bcast_slice(sm.st, kStageBytes, reinterpret_cast<unsigned char*>(sm.qs + n0), QD * 2, R, (q_end - n0) * 2);
      } else if (j == 1 || j == 3) {  // O-proj / down + residual
        const int nc = j == 1 ? no : nd, n0 = static_cast<int>(c) * nc;
        auto epi = [&](int cl, int r, float v, float) {
          if (r < R) stf[r * SF + cl] = sm.xs[r * D + n0 + cl] + v;
        };
        if (j == 1)
          slab_gemv<RP, false>(W, no, QD, sm, D, nullptr, sm.os, R, epi);
        else
          slab_gemv<RP, false>(W, nd, FF, sm, D, nullptr, sm.hs, R, epi);
        __syncthreads();
        if (l == 1) sstamp(4 + j * 4);
        bcast_slice(sm.st, kStageBytes, reinterpret_cast<unsigned char*>(sm.xs + n0), D * 4, R, nc * 4);
      } else {  // gate/up + SwiGLU
        const int n0 = static_cast<int>(c) * ng;
        slab_gemv<RP, true>(W, ng, D, sm, D, P.g, nullptr, R, [&](int cl, int r, float v, float partner) {
          if (r >= R || (cl & 1)) return;
          stb[r * SB + cl / 2] = __float2bfloat16_rn(v / (1.0f + __expf(-v)) * partner);
        });
        __syncthreads();
        if (l == 1) sstamp(12);
        bcast_slice(sm.st, kStageBytes, reinterpret_cast<unsigned char*>(sm.hs + n0 / 2), FF * 2, R, ng);
      }
      __syncthreads();  // slot consumed, staging free
      if (l == 1) sstamp(5 + j * 4);
      if (threadIdx.x == 0 && s + 2 < nslab) {
        unsigned bytes;
        const bf16* src = slab_src(s + 2, &bytes);
        mbar_expect_tx(&sm.bar[slot], bytes);
        bulk_load(sm.w[slot], src, bytes, &sm.bar[slot]);
      }
      cluster_sync_all();  // this step's slices (and KV appends) are visible cluster-wide
      if (l == 1) sstamp(6 + j * 4);
      if (j == 0) {
        if (hd == 64)
          attention_step<64>(P, l, R, sm, c);
        else
          attention_step<128>(P, l, R, sm, c);
        if (l == 1) sstamp(20);
        cluster_sync_all();
        if (l == 1) sstamp(21);
      }
    }
  }
}

__global__ void __launch_bounds__(NT, 1) small_forward_kernel(const SmallParams P) {
  extern __shared__ unsigned char smem_raw[];
  const Sm sm = carve(smem_raw, P);
  const unsigned c = cluster_rank();
  const int D = P.D, QD = P.nh * P.hd, FF = P.ffn;
  const int qkv_cols = (P.nh + 2 * P.nkv) * P.hd;
  const int nq = qkv_cols / CS;
  if (threadIdx.x == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // weights do not depend on the previous kernel: first two slabs now
    const bf16* base = P.w0;
    const unsigned b0 = nq * D * 2, b1 = (D / CS) * QD * 2;
    mbar_expect_tx(&sm.bar[0], b0);
    bulk_load(sm.w[0], base + static_cast<long long>(c) * nq * D, b0, &sm.bar[0]);
    mbar_expect_tx(&sm.bar[1], b1);
    bulk_load(sm.w[1], base + P.off_o + static_cast<long long>(c) * (D / CS) * QD, b1, &sm.bar[1]);
  }
  (void)FF;
  sstamp(0);
  pdl_launch_dependents();
  pdl_wait();
  sstamp(1);
  const int R = __ldg(P.meta);
  // embedding rows -> local x replica
  for (int i = threadIdx.x; i < R * (D / 8); i += NT) {
    const int r = i / (D / 8), k = (i % (D / 8)) * 8;
    int tok = P.rows[r].tok;
    if (tok < 0) tok = __ldcg(P.out_tok_read - 1 - tok);
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(P.emb + static_cast<long long>(tok) * D + k), f);
    float4* dst = reinterpret_cast<float4*>(sm.xs + r * D + k);
    dst[0] = make_float4(f[0], f[1], f[2], f[3]);
    dst[1] = make_float4(f[4], f[5], f[6], f[7]);
  }
  __syncthreads();
  cluster_sync_all();  // every CTA of the cluster is running before remote writes start
  sstamp(2);
  if (R <= 4)
    run_layers<4>(P, sm, c, R);
  else if (R <= 8)
    run_layers<8>(P, sm, c, R);
  else
    run_layers<16>(P, sm, c, R);
  sstamp(22);
  if (c == 0)
    for (int i = threadIdx.x; i < R * D; i += NT) P.x_out[i] = sm.xs[i];
}

}  // namespace

void small_forward_debug_trace(unsigned long long* buf) { cudaMemcpyToSymbol(g_small_trace, &buf, sizeof(buf)); }

int small_forward_smem(const SmallParams& p) {
  const int QD = p.nh * p.hd;
  return 128 + 2 * kSlot + RMAX * p.D * 4 + RMAX * p.ffn * 2 + 2 * RMAX * QD * 2 + RMAX * kStageBytes + 4 * p.hd * 4 +
         NW * 4 * p.hd * 4 + 2 * NW * 4 * 4 + 32 + RMAX * 4 + 64;
}

bool small_forward_supported(const SmallParams& p) {
  const int qkv_cols = (p.nh + 2 * p.nkv) * p.hd;
  const int QD = p.nh * p.hd;
  if (p.hd != 64 && p.hd != 128) return false;
  if (p.nh % p.nkv || p.nh / p.nkv > 4) return false;
  // per-CTA column slabs: multiples of 16 columns (column groups, 16-byte slices)
  if (qkv_cols % (16 * CS) || p.D % (16 * CS) || (2 * p.ffn) % (16 * CS)) return false;
  if (p.D % 256 || QD % 256 || p.ffn % 256) return false;  // K loops step 256 per warp
  if ((p.D / CS) * 4 > kStageBytes || (2 * p.ffn / CS) > kStageBytes / 2 || (qkv_cols / CS) * 2 > kStageBytes) return false;
  if ((p.nh / p.nkv) * p.hd * 2 > kStageBytes) return false;
  const long long slabs[4] = {static_cast<long long>(qkv_cols / CS) * p.D * 2, static_cast<long long>(p.D / CS) * QD * 2,
                              static_cast<long long>(2 * p.ffn / CS) * p.D * 2,
                              static_cast<long long>(p.D / CS) * p.ffn * 2};
  for (long long b : slabs)
    if (b > kSlot || b % 16) return false;
  if (small_forward_smem(p) > 227 * 1024) return false;
  int n = 0;
  cudaFuncSetAttribute(small_forward_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(small_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, small_forward_smem(p));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = small_forward_smem(p);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&n, small_forward_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

void small_forward(const SmallParams& p, cudaStream_t st) {
  const int smem = small_forward_smem(p);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CS);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&cfg, small_forward_kernel, p);
}

}  // namespace moa::k
