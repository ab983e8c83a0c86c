// Persistent decode forward ("megakernel") for ticks of <= 16 rows of one
// model: the whole forward -- embedding, every layer's QKV / attention /
// O-proj / gate-up / down, and the LM head with greedy statistics -- in ONE
// launch of one CTA per SM.
//
// Why: a decode tick of a 1B agent is a stream of ~2 GB of weights through
// ~80 small GEMVs; as separate kernels every GEMV pays its launch, TMEM/
// barrier setup, first-byte latency and split-K tail, so the tick ran at ~15%
// of HBM bandwidth (profiles/r02).  Here the weight stream never waits on
// activations:
//
//   warp 6  (TMA producer)  streams this CTA's weight tiles for every phase of
//                           the forward, in order, into an smem ring; it only
//                           waits for free ring stages.
//   warp 7  (MMA issuer)    one thread: tcgen05.mma, swap-AB
//                           D[128 weight rows][16 rows] += W_tile . X_tile^T,
//                           fp32 accumulators double-buffered in TMEM.
//   warps 0-5 (workers)     wait for the previous phase (grid barrier, one
//                           poller per CTA), stage the phase's activation
//                           k-tiles in smem (RMSNorm applied on the fly, bf16,
//                           128B-swizzled K-major = the layout TMA would
//                           write), run the attention and embedding phases;
//                           warps 0-3 also run the GEMV epilogues: tcgen05.ld
//                           (thread = weight row), split-K partials with a
//                           deterministic last-arriver reduction, fused RoPE +
//                           KV append / residual + row sum-of-squares /
//                           SwiGLU / LM-head greedy statistics.
//
// The ring absorbs the grid barriers and the attention phase: while the
// workers wait, the producer keeps prefetching the next phase's weights.
//
// Work split (host-computed, decode_mk_plan): a GEMV phase is T weight tiles
// (128 rows) x KT k-tiles (64); its U = T*KT units are split into G contiguous
// ranges (CTA c owns [c*U/G, (c+1)*U/G)), each cut into per-tile segments.
// Partial sums are combined in CTA order by the last CTA to finish the tile,
// so results depend only on (N, K, G) -- never on timing or on which rows
// share the tick.
//
// Intra-kernel produced data (x, q, o, h, KV at the new position, partials)
// is read with ld.global.cg (L2): L1 is not coherent across SMs.
#include <cfloat>
#include <climits>
#include <cstdio>
#include <type_traits>
#include <vector>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace moa::k {

namespace {

using namespace tc;

constexpr int kN = kMkRows;  // activation rows = MMA N
constexpr int kM = 128;      // weight rows per tile = MMA M
constexpr int kBK = 64;      // K per unit (one 128-byte swizzle row)
constexpr int kMaxStages = 16;
constexpr int kTileW = kM * kBK * 2;  // 16 KB
constexpr int kTileX = kN * kBK * 2;  // 2 KB
constexpr int kThreads = 256;  // 8 warps: 255 registers per thread (10 warps would cap at 168)
constexpr int kAttnWarps = 6;  // workers: warps 0-5
constexpr int kWorkers = kAttnWarps * 32;
constexpr int kQsFloats = kMkMaxGroupDims;  // per worker warp: HPG * hd fp32 q values
constexpr int kSmemBudget = 227 * 1024;
constexpr int kSmemFixed = 1024 + kAttnWarps * kQsFloats * 4 + 5 * static_cast<int>(sizeof(MkCtaPlan)) + 2048;
constexpr std::uint32_t kIdesc = idesc_bf16(kM, kN);
constexpr int kMinUnits = 4;  // k-tiles per CTA per GEMV phase, at least (decode_mk_plan)

enum PhaseKind { PK_EMBED = 0, PK_QKV, PK_ATTN, PK_O, PK_GU, PK_DOWN, PK_LM, PK_LMX };
enum XSrc { XS_NORM = 0, XS_NORM_SEL = 1, XS_BF16 = 2 };

__device__ __forceinline__ int phase_kind(int p, int L) {
  if (p == 0) return PK_EMBED;
  if (p == 1 + 5 * L) return PK_LM;
  if (p == 2 + 5 * L) return PK_LMX;
  return PK_QKV + (p - 1) % 5;
}

// GEMV shape index into the plan table: QKV 0, O 1, GU 2, DOWN 3, LM 4
__device__ __forceinline__ int shape_of(int kind) {
  return kind == PK_QKV ? 0 : kind == PK_O ? 1 : kind == PK_GU ? 2 : kind == PK_DOWN ? 3 : 4;
}

struct Gemv {
  int map, N, K, epi, xsrc, layer;
  const bf16* xb;  // XS_BF16 source [rows][K]
};

__device__ __forceinline__ Gemv gemv_of(const MkParams& P, int p) {
  const int kind = phase_kind(p, P.L);
  const int l = (p - 1) / 5;
  Gemv g{};
  switch (kind) {
    case PK_QKV: g = Gemv{4 * l + 0, (P.nh + 2 * P.nkv) * P.hd, P.D, kEpiQkv, XS_NORM, l, nullptr}; break;
    case PK_O: g = Gemv{4 * l + 1, P.D, P.nh * P.hd, kEpiResidual, XS_BF16, l, P.o}; break;
    case PK_GU: g = Gemv{4 * l + 2, 2 * P.ffn, P.D, kEpiSwiGlu, XS_NORM, l, nullptr}; break;
    case PK_DOWN: g = Gemv{4 * l + 3, P.D, P.ffn, kEpiResidual, XS_BF16, l, P.h}; break;
    case PK_LM: g = Gemv{4 * P.L, P.V, P.D, kEpiLmStats, XS_NORM_SEL, P.L, nullptr}; break;
    default: break;
  }
  return g;
}

// ---- synchronisation helpers (bounded spins: a broken invariant traps
// instead of hanging the GPU) ----
__device__ __noinline__ void spin_timeout() {
  printf("decode_mk: spin timeout (block %d thread %d)\n", blockIdx.x, threadIdx.x);
  __trap();
}

__device__ __forceinline__ void mbar_wait_g(std::uint64_t* bar, std::uint32_t parity) {
  std::uint32_t ok = 0;
  const long long t0 = clock64();
  while (true) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > (1LL << 34)) spin_timeout();  // ~8 s
  }
}


__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Grid barrier over phases.  gbar[0] is a monotonically increasing arrival
// counter (wrap-safe compares), gbar[1] its value at the start of this launch
// (written by the previous launch's last arrival).  Every CTA adds 1 after
// finishing phase p; phase p is complete when gbar[0] - base >= (p + 1) * G.
// One thread per CTA polls (with back-off, so G pollers do not saturate the
// counter's L2 slice) and releases the CTA's workers through a named barrier;
// a CTA only arrives at p after observing p - 1, so counts cannot run ahead.
__device__ __forceinline__ void poll_phase(const unsigned* gbar, unsigned base, int p, int G) {
  if (p < 0) return;
  const unsigned target = static_cast<unsigned>(p + 1) * G;
  const long long t0 = clock64();
  while (static_cast<int>(ld_relaxed(gbar) - base - target) < 0) {
    __nanosleep(32);
    if (clock64() - t0 > (1LL << 34)) spin_timeout();
  }
  fence_acq_rel();
}

__device__ __forceinline__ void arrive_phase(unsigned* gbar, unsigned base, int p, int G, int P_total) {
  if (p != P_total - 1) {
    red_add_release(gbar, 1u);  // release: the CTA's writes (ordered before by bar.sync) become visible first
    return;
  }
  const unsigned prev = atom_add_acq_rel(gbar, 1u);
  if (prev - base == static_cast<unsigned>(P_total) * G - 1) gbar[1] = base + static_cast<unsigned>(P_total) * G;
}

__device__ __forceinline__ void stamp(const MkParams& P, int p, int ev) {
  if (P.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    P.trace[(static_cast<long long>(p) * gridDim.x + blockIdx.x) * 8 + ev] = t;
  }
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
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
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
  return LmStat{__shfl_xor_sync(0xffffffffu, s.m, off), __shfl_xor_sync(0xffffffffu, s.s, off),
                __shfl_xor_sync(0xffffffffu, s.t, off), __shfl_xor_sync(0xffffffffu, s.idx, off)};
}

struct Smem {
  unsigned char* w;   // [stages][kTileW] weight ring
  unsigned char* xs;  // [xs_kt][kTileX] activation staging of the current phase (slot = kt % xs_kt)
  std::uint64_t* full;
  std::uint64_t* empty;
  std::uint64_t* acc_full;   // [2]
  std::uint64_t* acc_empty;  // [2]
  std::uint64_t* x_ready;    // staging written (workers -> MMA)
  std::uint32_t* tmem_slot;
  float* qs;        // [kAttnWarps][kQsFloats]
  MkCtaPlan* plan;  // [5] this CTA's segments per GEMV shape
  float* inv;       // [kN]
  float* red;       // [4][kN] (epilogue row reductions)
  LmStat* lmred;    // [4][kN]
  int* flag;        // [4]
};

__device__ __forceinline__ Smem carve(unsigned char* raw, int stages, int xs_kt) {
  unsigned char* p =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(raw) + 1023) & ~std::uintptr_t(1023));
  Smem s;
  s.w = p;
  p += stages * kTileW;
  s.xs = p;
  p += xs_kt * kTileX;
  s.qs = reinterpret_cast<float*>(p);
  p += kAttnWarps * kQsFloats * 4;
  s.plan = reinterpret_cast<MkCtaPlan*>(p);
  p += 5 * sizeof(MkCtaPlan);
  s.full = reinterpret_cast<std::uint64_t*>(p);
  s.empty = s.full + kMaxStages;
  s.acc_full = s.empty + kMaxStages;
  s.acc_empty = s.acc_full + 2;
  s.x_ready = s.acc_empty + 2;
  s.tmem_slot = reinterpret_cast<std::uint32_t*>(s.x_ready + 1);
  s.inv = reinterpret_cast<float*>(s.tmem_slot + 4);
  s.red = s.inv + kN;
  s.lmred = reinterpret_cast<LmStat*>(s.red + 4 * kN);
  s.flag = reinterpret_cast<int*>(s.lmred + 4 * kN);
  return s;
}

// ---------------- epilogues (thread = weight row n, v[r] = row r) ----------------

__device__ __forceinline__ void epi_store(const MkParams& P, const Gemv& g, int n, int R, float (&v)[kN], const Smem& sm, int tile) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  (void)lane;
  switch (g.epi) {
    case kEpiResidual: {
      // x[r][n] += v; per-row sum of squares of this tile's 128 new values
#pragma unroll
      for (int r = 0; r < kN; ++r) {
        float nv = 0.f;
        if (r < R && n < g.N) {
          float* xp = P.x + static_cast<long long>(r) * P.D + n;
          nv = __ldcg(xp) + v[r];
          __stcg(xp, nv);
        }
        const float ss = warp_sum(nv * nv);
        if ((threadIdx.x & 31) == 0) sm.red[warp * kN + r] = ss;
      }
      named_sync(2, 128);
      if (threadIdx.x < kN) {
        const int r = threadIdx.x;
        const float ss = (sm.red[r] + sm.red[kN + r]) + (sm.red[2 * kN + r] + sm.red[3 * kN + r]);
        __stcg(P.ssq + r * (P.D / kM) + tile, ss);
      }
      named_sync(2, 128);
      break;
    }
    case kEpiSwiGlu: {
#pragma unroll
      for (int r = 0; r < kN; ++r) {
        const float x = v[r];
        const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
        if (r < R && n < g.N && !(n & 1))
          P.h[static_cast<long long>(r) * P.ffn + n / 2] = __float2bfloat16_rn(x / (1.0f + __expf(-x)) * partner);
      }
      break;
    }
    case kEpiQkv: {
      const int hd = P.hd, half = hd / 2, qk_cols = (P.nh + P.nkv) * hd;
      const long long loff = P.layer_stride * g.layer;
#pragma unroll
      for (int r = 0; r < kN; ++r) {
        const float x = v[r];
        const float partner = __shfl_xor_sync(0xffffffffu, x, 1);
        if (r >= R || n >= g.N) continue;
        const RowDesc rd = P.rows[r];
        if (n < qk_cols) {
          if (n & 1) continue;
          const int head = n / hd, e = (n % hd) / 2;
          const float2 cs = P.rope[static_cast<long long>(rd.pos) * half + e];
          const float y0 = __fsub_rn(__fmul_rn(x, cs.x), __fmul_rn(partner, cs.y));
          const float y1 = __fadd_rn(__fmul_rn(partner, cs.x), __fmul_rn(x, cs.y));
          bf16* dst = head < P.nh ? P.q + (static_cast<long long>(r) * P.nh + head) * hd
                                  : P.kpool + rd.kv * P.kv_stride + loff +
                                        (static_cast<long long>(head - P.nh) * P.max_ctx + rd.pos) * hd;
          dst[e] = __float2bfloat16_rn(y0);
          dst[e + half] = __float2bfloat16_rn(y1);
        } else {
          const int vc = n - qk_cols, kh = vc / hd, e = vc % hd;
          P.vpool[rd.kv * P.kv_stride + loff + (static_cast<long long>(kh) * P.max_ctx + rd.pos) * hd + e] =
              __float2bfloat16_rn(x);
        }
      }
      break;
    }
    case kEpiLmStats: {
      // per logits row: greedy statistics over this tile's 128 vocab entries
      // (merged over all tiles in the LMX phase, fixed order)
      const int warp_ = threadIdx.x >> 5, ln = threadIdx.x & 31;
      const LmStat none{-INFINITY, 0.f, 0.f, 0x7fffffff};
      const int ntiles = (P.V + kM - 1) / kM;
#pragma unroll
      for (int r = 0; r < kN; ++r) {
        if (r >= R) break;
        const bool ok = n < P.V;
        if (ok && P.logits) P.logits[static_cast<long long>(r) * P.V + n] = v[r];
        LmStat st = ok ? LmStat{v[r], 1.f, 0.f, n} : none;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const LmStat o = shfl_stat(st, off);
          st = (ln & off) ? stat_merge(o, st) : stat_merge(st, o);
        }
        if (ln == 0) sm.lmred[warp_ * kN + r] = st;
      }
      named_sync(2, 128);
      if (threadIdx.x < R) {
        LmStat st = sm.lmred[threadIdx.x];
        for (int w = 1; w < 4; ++w) st = stat_merge(st, sm.lmred[w * kN + threadIdx.x]);
        __stcg(reinterpret_cast<float4*>(P.lm_part + static_cast<long long>(threadIdx.x) * ntiles + tile),
               make_float4(st.m, st.s, st.t, __int_as_float(st.idx)));
      }
      named_sync(2, 128);
      break;
    }
    default:
      break;
  }
}

// Unit = (row, kv head, KS-key split): the group's q heads share one read of
// the split's K and V.  K: TPK lanes per key, each holding 64 dims of the
// key's row; V: lane owns HD/32 output dims of every key.
template <int HD>
__device__ __noinline__ void attention_phase(const MkParams& P, int layer, int R, const Smem& sm, int G) {
  constexpr int TPK = HD / 64;      // lanes per key
  constexpr int KS = 32 / TPK;      // keys per unit
  constexpr int E = HD / 32;        // output dims per lane
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int key = lane / TPK, part = lane % TPK;  // this lane's key in the split, and which 64 dims
  const int hpg = P.nh / P.nkv;
  const long long loff = P.layer_stride * layer;
  float* qs = sm.qs + warp * kQsFloats;
  int total = 0;
  for (int r = 0; r < R; ++r) total += P.nkv * ((P.rows[r].pos + KS) / KS);
  const float scale = rsqrtf(static_cast<float>(HD));
  for (int u = blockIdx.x * kAttnWarps + warp; u < total; u += G * kAttnWarps) {
    int r = 0, rem = u, ns = 0;
    for (; r < R; ++r) {
      ns = (P.rows[r].pos + KS) / KS;
      if (rem < P.nkv * ns) break;
      rem -= P.nkv * ns;
    }
    const RowDesc rd = P.rows[r];
    const int g = rem / ns, s = rem % ns, n = rd.pos + 1;
    const bf16* K = P.kpool + rd.kv * P.kv_stride + loff + static_cast<long long>(g) * P.max_ctx * HD;
    const bf16* V = P.vpool + rd.kv * P.kv_stride + loff + static_cast<long long>(g) * P.max_ctx * HD;
    const int j0 = s * KS;
    const int jk = j0 + key;
    // issue this unit's K and V loads before any compute
    uint4 kk[8];
#pragma unroll
    for (int v = 0; v < 8; ++v)
      kk[v] = jk < n ? __ldcg(reinterpret_cast<const uint4*>(K + static_cast<long long>(jk) * HD + part * 64) + v)
                     : make_uint4(0, 0, 0, 0);
    using VT = typename std::conditional<E == 2, unsigned, uint2>::type;
    VT vv[KS];
#pragma unroll
    for (int jj = 0; jj < KS; ++jj) {
      const int j = j0 + jj;
      if (j < n)
        vv[jj] = __ldcg(reinterpret_cast<const VT*>(V + static_cast<long long>(j) * HD + lane * E));
      else
        vv[jj] = VT{};
    }
    for (int i = lane; i < hpg * HD; i += 32) {
      const int h = g * hpg + i / HD;
      qs[i] = __bfloat162float(__ldcg(P.q + (static_cast<long long>(r) * P.nh + h) * HD + (i % HD)));
    }
    __syncwarp();
    const int nsplit = ns;
    for (int hh = 0; hh < hpg; ++hh) {
      const float* qh = qs + hh * HD + part * 64;
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
      const float sc = jk < n ? d * scale : -INFINITY;
      const float m = warp_max(sc);
      const float pk = jk < n ? __expf(sc - m) : 0.f;
      const float l = warp_sum(part == 0 ? pk : 0.f);
      float acc[E];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = 0.f;
#pragma unroll
      for (int jj = 0; jj < KS; ++jj) {
        const float pj = __shfl_sync(0xffffffffu, pk, jj * TPK);
        if constexpr (E == 2) {
          const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj]));
          acc[0] = fmaf(pj, f.x, acc[0]);
          acc[1] = fmaf(pj, f.y, acc[1]);
        } else {
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].x));
          const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[jj].y));
          acc[0] = fmaf(pj, f0.x, acc[0]);
          acc[1] = fmaf(pj, f0.y, acc[1]);
          acc[2] = fmaf(pj, f1.x, acc[2]);
          acc[3] = fmaf(pj, f1.y, acc[3]);
        }
      }
      const int head = g * hpg + hh;
      if (nsplit == 1) {
        bf16* orow = P.o + (static_cast<long long>(r) * P.nh + head) * HD + lane * E;
#pragma unroll
        for (int e = 0; e < E; ++e) orow[e] = __float2bfloat16_rn(acc[e] / l);
      } else {
        float* pp = P.attn_ws + ((static_cast<long long>(r) * P.nh + head) * P.attn_nsplit_max + s) * (2 + HD);
        if (lane == 0) {
          __stcg(pp, m);
          __stcg(pp + 1, l);
        }
#pragma unroll
        for (int e = 0; e < E; ++e) __stcg(pp + 2 + lane * E + e, acc[e]);
      }
    }
    if (nsplit > 1) {
      __syncwarp();
      int last = 0;
      if (lane == 0)
        last = atom_add_acq_rel(reinterpret_cast<unsigned*>(P.attn_cnt + r * P.nkv + g), 1u) ==
               static_cast<unsigned>(nsplit - 1);
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        for (int hh = 0; hh < hpg; ++hh) {
          const int head = g * hpg + hh;
          const float* pr = P.attn_ws + (static_cast<long long>(r) * P.nh + head) * P.attn_nsplit_max * (2 + HD);
          // split statistics: lane t holds split t (+32k), combined by shuffles
          float mt = -INFINITY, lt = 0.f;
          for (int t = lane; t < nsplit; t += 32) {
            const float m2 = __ldcg(pr + t * (2 + HD)), l2 = __ldcg(pr + t * (2 + HD) + 1);
            const float mn = fmaxf(mt, m2);
            lt = lt * __expf(mt - mn) + l2 * __expf(m2 - mn);
            mt = mn;
          }
          const float M = warp_max(mt);
          const float Lsum = warp_sum(mt == -INFINITY ? 0.f : lt * __expf(mt - M));
          float acc[E];
#pragma unroll
          for (int e = 0; e < E; ++e) acc[e] = 0.f;
          for (int t0 = 0; t0 < nsplit; t0 += 4) {
            float pv[4][E], wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int t = t0 + u;
              wv[u] = 0.f;
              if (t < nsplit) {
                wv[u] = __expf(__ldcg(pr + t * (2 + HD)) - M);
#pragma unroll
                for (int e = 0; e < E; ++e) pv[u][e] = __ldcg(pr + t * (2 + HD) + 2 + lane * E + e);
              } else {
#pragma unroll
                for (int e = 0; e < E; ++e) pv[u][e] = 0.f;
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int e = 0; e < E; ++e) acc[e] = fmaf(wv[u], pv[u][e], acc[e]);
          }
          bf16* orow = P.o + (static_cast<long long>(r) * P.nh + head) * HD + lane * E;
#pragma unroll
          for (int e = 0; e < E; ++e) orow[e] = __float2bfloat16_rn(acc[e] / Lsum);
        }
        if (lane == 0) __stcg(P.attn_cnt + r * P.nkv + g, 0);
      }
    }
    __syncwarp();
  }
}

// LM merge: row r's tile statistics (written by the LM phase) merged in tile
// order by one warp -> greedy token, logprob, entropy.
__device__ __noinline__ void lm_merge_phase(const MkParams& P, int Rl, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntiles = (P.V + kM - 1) / kM;
  const LmStat none{-INFINITY, 0.f, 0.f, 0x7fffffff};
  for (int r = blockIdx.x * kAttnWarps + warp; r < Rl; r += G * kAttnWarps) {
    LmStat st = none;
    const float4* pr = reinterpret_cast<const float4*>(P.lm_part + static_cast<long long>(r) * ntiles);
    for (int b0 = lane; b0 < ntiles; b0 += 32 * 8) {
      float4 raw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + 32 * u;
        raw[u] = b < ntiles ? __ldcg(pr + b) : make_float4(-INFINITY, 0.f, 0.f, __int_as_float(0x7fffffff));
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
      const int oi = P.out_idx[r];
      const float ls = logf(st.s);
      P.out_tok[oi] = st.idx;
      P.out_lp[oi] = -ls;
      P.out_ent[oi] = ls - st.t / st.s;
    }
  }
}

// embedding rows -> x (fp32) and the per-tile sums of squares for layer 0's norm
__device__ __noinline__ void embed_phase(const MkParams& P, int R, int G) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tiles = P.D / kM;
  for (int u = blockIdx.x * kAttnWarps + warp; u < R * tiles; u += G * kAttnWarps) {
    const int r = u / tiles, t = u % tiles;
    int tok = P.rows[r].tok;
    if (tok < 0) tok = __ldcg(P.out_tok_read - 1 - tok);
    const int c = t * kM + lane * 4;
    const uint2 raw = *reinterpret_cast<const uint2*>(P.emb + static_cast<long long>(tok) * P.D + c);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
    __stcg(reinterpret_cast<float4*>(P.x + static_cast<long long>(r) * P.D + c), make_float4(a.x, a.y, b.x, b.y));
    const float ss = warp_sum(a.x * a.x + a.y * a.y + b.x * b.x + b.y * b.y);
    if (lane == 0) __stcg(P.ssq + r * tiles + t, ss);
  }
}

// Stage one GEMV phase's activation k-tiles into smem (workers, warps 0-5):
// rows < `rows` only (MMA columns are independent, stale rows only feed
// ignored outputs); the norm statistics and the activations load in the same
// round trip.  Out of line: its own register allocation (no spills).
__device__ __noinline__ void stage_activations(const MkParams& P, const Gemv g, const MkCtaPlan& pl, int rows,
                                               const Smem& sm) {
  const int wt = threadIdx.x;
        constexpr int U = 4;
        const int nchunk = pl.nkt * rows * 8;  // (k-tile, row, 16-byte chunk)
        float ssq_part = 0.f;
        if (g.xsrc != XS_BF16 && wt < kN * 8) {  // 8 threads per row sum the row's tile partials
          const int r = wt >> 3, j = wt & 7;
          if (r < rows) {
            const int src = g.xsrc == XS_NORM_SEL ? __ldg(P.sel + r) : r;
            const int tiles = P.D / kM;
            for (int t = j; t < tiles; t += 8) ssq_part += __ldcg(P.ssq + src * tiles + t);
          }
        }
        uint4 out[U];
        float4 ra[U], rb[U];
        int dst[U], col[U], rr[U];
        for (int base = 0; base < nchunk; base += kWorkers * U) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int ch = base + u * kWorkers + wt;
            dst[u] = -1;
            if (ch >= nchunk) continue;
            const int si = ch / (rows * 8), r = (ch >> 3) % rows, cc = ch & 7;
            const int kt = pl.kt[si];
            rr[u] = r;
            dst[u] = (kt % P.xs_kt) * kTileX + r * 128 + ((cc ^ (r & 7)) * 16);
            col[u] = kt * kBK + cc * 8;
            if (g.xsrc == XS_BF16) {
              out[u] = __ldcg(reinterpret_cast<const uint4*>(g.xb + static_cast<long long>(r) * g.K + col[u]));
            } else {
              const int src = g.xsrc == XS_NORM_SEL ? __ldg(P.sel + r) : r;
              const float4* xp = reinterpret_cast<const float4*>(P.x + static_cast<long long>(src) * P.D + col[u]);
              ra[u] = __ldcg(xp);
              rb[u] = __ldcg(xp + 1);
            }
          }
          if (g.xsrc != XS_BF16) {
            if (base == 0) {  // finish the norm statistics: 8 partials per row -> inv
              float t = ssq_part;
              t += __shfl_xor_sync(0xffffffffu, t, 1);
              t += __shfl_xor_sync(0xffffffffu, t, 2);
              t += __shfl_xor_sync(0xffffffffu, t, 4);
              if (wt < kN * 8 && (wt & 7) == 0) sm.inv[wt >> 3] = 1.0f / sqrtf(t / static_cast<float>(P.D) + P.eps);
              named_sync(1, kWorkers);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (dst[u] < 0) continue;
              const float iv = sm.inv[rr[u]];
              const float4 ga = __ldg(reinterpret_cast<const float4*>(P.g + col[u]));
              const float4 gb = __ldg(reinterpret_cast<const float4*>(P.g + col[u] + 4));
              __align__(16) bf16 o8[8];
              o8[0] = __float2bfloat16_rn(ra[u].x * iv * ga.x);
              o8[1] = __float2bfloat16_rn(ra[u].y * iv * ga.y);
              o8[2] = __float2bfloat16_rn(ra[u].z * iv * ga.z);
              o8[3] = __float2bfloat16_rn(ra[u].w * iv * ga.w);
              o8[4] = __float2bfloat16_rn(rb[u].x * iv * gb.x);
              o8[5] = __float2bfloat16_rn(rb[u].y * iv * gb.y);
              o8[6] = __float2bfloat16_rn(rb[u].z * iv * gb.z);
              o8[7] = __float2bfloat16_rn(rb[u].w * iv * gb.w);
              out[u] = *reinterpret_cast<const uint4*>(o8);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (dst[u] >= 0) *reinterpret_cast<uint4*>(sm.xs + dst[u]) = out[u];
        }
}

// The GEMV epilogues of one phase for this CTA's segments (warps 0-3):
// tcgen05.ld, split-K partials + deterministic last-arriver reduction, fused
// epilogue.  Returns the running segment counter.  Out of line (registers).
__device__ __noinline__ int gemv_epilogues(const MkParams& P, const Gemv g, const MkCtaPlan& pl, int rows,
                                           const Smem& sm, std::uint32_t tmem, int sc, int c, int p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int i = 0; i < pl.nseg; ++i) {
        const MkSeg s = pl.seg[i];
        const int b = sc & 1;
        mbar_wait_g(&sm.acc_full[b], (sc >> 1) & 1);
        tc_fence_after();
        if (threadIdx.x == 0 && i == 0) stamp(P, p, 3);
        float v[kN];
        tmem_ld16(tmem + b * kN + (static_cast<std::uint32_t>(warp * 32) << 16), v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.acc_empty[b]);
        ++sc;
        const int n = s.t * kM + warp * 32 + lane;
        const int nseg = s.c_last - s.c_first + 1;
        if (nseg > 1) {
          // split-K: partial of this CTA; the last arriver sums all in CTA order
          float4* pw = reinterpret_cast<float4*>(P.ws + ((static_cast<long long>(c) * 2 + s.slot_self) * kM +
                                                         warp * 32 + lane) * kN);
#pragma unroll
          for (int j = 0; j < kN / 4; ++j) __stcg(pw + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
          named_sync(2, 128);
          if (threadIdx.x == 0)
            sm.flag[1] =
                atom_add_acq_rel(reinterpret_cast<unsigned*>(P.cnt + s.t), 1u) == static_cast<unsigned>(nseg - 1);
          named_sync(2, 128);
          if (!sm.flag[1]) continue;
#pragma unroll
          for (int j = 0; j < kN; ++j) v[j] = 0.f;
          // partials of 4 CTAs in flight per round trip, summed in CTA order
          for (int c0 = s.c_first; c0 <= s.c_last; c0 += 2) {
            float4 t4[2][kN / 4];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int cc = c0 + k;
              if (cc > s.c_last) break;
              const int slot = cc == s.c_first ? s.first_slot : 0;
              const float4* pr = reinterpret_cast<const float4*>(
                  P.ws + ((static_cast<long long>(cc) * 2 + slot) * kM + warp * 32 + lane) * kN);
#pragma unroll
              for (int j = 0; j < kN / 4; ++j) t4[k][j] = __ldcg(pr + j);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              if (c0 + k > s.c_last) break;
#pragma unroll
              for (int j = 0; j < kN / 4; ++j) {
                v[4 * j] += t4[k][j].x;
                v[4 * j + 1] += t4[k][j].y;
                v[4 * j + 2] += t4[k][j].z;
                v[4 * j + 3] += t4[k][j].w;
              }
            }
          }
          if (threadIdx.x == 0) __stcg(P.cnt + s.t, 0);
        }
        epi_store(P, g, n, rows, v, sm, s.t);
      }
  return sc;
}

// ---------------- the kernel ----------------

__global__ void __launch_bounds__(kThreads, 1) decode_mk_kernel(const MkParams P) {
  extern __shared__ unsigned char smem_raw[];
  const int stages = P.stages;
  const Smem sm = carve(smem_raw, stages, P.xs_kt);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  const int L = P.L;
  const int P_total = 3 + 5 * L;

  {  // this CTA's plan -> smem
    const int4* src = reinterpret_cast<const int4*>(P.plan + static_cast<long long>(c) * 5);
    int4* dst = reinterpret_cast<int4*>(sm.plan);
    for (int i = threadIdx.x; i < static_cast<int>(5 * sizeof(MkCtaPlan) / 16); i += kThreads) dst[i] = __ldg(src + i);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.acc_full[b], 1);
      mbar_init(&sm.acc_empty[b], 4);
    }
    mbar_init(sm.x_ready, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<32>(sm.tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *sm.tmem_slot;
  const int R = __ldg(P.meta);
  const int Rl = __ldg(P.meta + 1);
  const unsigned gbase = __ldcg(P.gbar + 1);

  if (warp == 6) {
    // ---------------- TMA weight producer: never waits on activations ----------------
    if (lane == 0) {
      stamp(P, 0, 5);
      const CUtensorMap* maps = static_cast<const CUtensorMap*>(P.maps);
      for (int i = 0; i < 4 * L + 1; ++i) prefetch_tmap(maps + i);
      int q = 0;
      for (int p = 1; p < P_total; ++p) {
        const int kind = phase_kind(p, L);
        if (kind == PK_ATTN || kind == PK_LMX) continue;
        const Gemv g = gemv_of(P, p);
        const CUtensorMap* map = maps + g.map;
        const MkCtaPlan& pl = sm.plan[shape_of(kind)];
        for (int i = 0; i < pl.nseg; ++i) {
          const MkSeg s = pl.seg[i];
          for (int kt = s.k0; kt < s.k1; ++kt, ++q) {
            const int st = q % stages;
            if (q >= stages) mbar_wait_g(&sm.empty[st], ((q / stages) - 1) & 1);
            if (i == 0 && kt == s.k0) stamp(P, p, 6);
            mbar_expect_tx(&sm.full[st], kTileW);
            tma_load_2d(sm.w + st * kTileW, map, &sm.full[st], kt * kBK, s.t * kM);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 7) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int q = 0, sc = 0, ph = 0;
      const std::uint32_t xs0 = smem_u32(sm.xs);
      for (int p = 1; p < P_total; ++p) {
        const int kind = phase_kind(p, L);
        if (kind == PK_ATTN || kind == PK_LMX) continue;
        const MkCtaPlan& pl = sm.plan[shape_of(kind)];
        if (pl.nseg == 0) continue;
        mbar_wait_g(sm.x_ready, ph & 1);  // this phase's activation staging is written
        ++ph;
        stamp(P, p, 2);
        for (int i = 0; i < pl.nseg; ++i) {
          const MkSeg s = pl.seg[i];
          const int b = sc & 1;
          if (sc >= 2) mbar_wait_g(&sm.acc_empty[b], ((sc >> 1) - 1) & 1);
          tc_fence_after();
          const std::uint32_t d = tmem + b * kN;
          for (int kt = s.k0; kt < s.k1; ++kt, ++q) {
            const int st = q % stages;
            mbar_wait_g(&sm.full[st], (q / stages) & 1);
            tc_fence_after();
            const std::uint32_t w0 = smem_u32(sm.w + st * kTileW), x0 = xs0 + (kt % P.xs_kt) * kTileX;
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16(d, umma_desc(w0 + k * 32), umma_desc(x0 + k * 32), kIdesc, (kt > s.k0 || k) ? 1u : 0u);
            umma_commit(&sm.empty[st]);
          }
          umma_commit(&sm.acc_full[b]);
          ++sc;
        }
        stamp(P, p, 7);
      }
    }
    __syncwarp();
  } else {
    // ---------------- workers, warps 0-5 ----------------
    const int wt = threadIdx.x;  // 0..191
    const bool epi = warp < 4;
    int sc = 0;
    for (int p = 0; p < P_total; ++p) {
      const int kind = phase_kind(p, L);
      if (wt == 0) {
        poll_phase(P.gbar, gbase, p - 1, G);
        stamp(P, p, 0);
      }
      named_sync(1, kWorkers);
      if (kind == PK_EMBED || kind == PK_ATTN || kind == PK_LMX) {
        if (kind == PK_EMBED)
          embed_phase(P, R, G);
        else if (kind == PK_LMX)
          lm_merge_phase(P, Rl, G);
        else if (P.hd == 64)
          attention_phase<64>(P, (p - 1) / 5, R, sm, G);
        else
          attention_phase<128>(P, (p - 1) / 5, R, sm, G);
        named_sync(1, kWorkers);
        if (wt == 0) {
          stamp(P, p, 4);
          arrive_phase(P.gbar, gbase, p, G, P_total);
        }
        continue;
      }
      const Gemv g = gemv_of(P, p);
      const MkCtaPlan& pl = sm.plan[shape_of(kind)];
      const int rows = kind == PK_LM ? Rl : R;
      if (pl.nseg > 0) {
        stage_activations(P, g, pl, rows, sm);
        fence_proxy_async_smem();
        named_sync(1, kWorkers);
        if (wt == 0) {
          mbar_arrive(sm.x_ready);
          stamp(P, p, 1);
        }
      }
      if (!epi) continue;
      // ---------------- epilogue (warps 0-3) ----------------
      sc = gemv_epilogues(P, g, pl, rows, sm, tmem, sc, c, p);
      named_sync(2, 128);
      if (threadIdx.x == 0) {
        stamp(P, p, 4);
        arrive_phase(P.gbar, gbase, p, G, P_total);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<32>(tmem);
}

}  // namespace

long long decode_mk_ws_floats(int grid) { return static_cast<long long>(grid) * 2 * kM * kN; }

int decode_mk_attn_splits(int hd, int max_ctx) {
  const int ks = hd == 64 ? 32 : 16;
  return (max_ctx + ks - 1) / ks;
}

bool decode_mk_supported(int d, int nh, int nkv, int hd, int ffn) {
  const int hpg = nh / nkv;
  return (hd == 64 || hd == 128) && d % kM == 0 && (nh * hd) % kBK == 0 && ffn % kBK == 0 && d % kBK == 0 &&
         hpg * hd <= kQsFloats;
}

// Host-computed static partition (see the header comment): per GEMV shape and
// CTA, its segments and the distinct k-tiles it stages; the smallest staging
// (slots = kt % xs_kt) with no collision inside any CTA's k-tile set; the ring
// depth the remaining shared memory allows.  false: no feasible plan.
bool decode_mk_plan(const MkParams& p, int grid, std::vector<MkCtaPlan>* plan, int* xs_kt, int* stages,
                    int* smem_bytes) {
  struct Ph {
    int N, K;
  };
  const Ph phases[5] = {{(p.nh + 2 * p.nkv) * p.hd, p.D}, {p.D, p.nh * p.hd}, {2 * p.ffn, p.D}, {p.D, p.ffn}, {p.V, p.D}};
  plan->assign(static_cast<std::size_t>(grid) * 5, MkCtaPlan{});
  for (int sh = 0; sh < 5; ++sh) {
    const long long T = (phases[sh].N + kM - 1) / kM, KT = phases[sh].K / kBK, U = T * KT;
    // CTAs used: at most one per kMinUnits units, so a small phase is not
    // shredded into 1-unit split-K pieces whose reduction costs more than
    // streaming the extra units
    const long long Ge = std::max<long long>(1, std::min<long long>(grid, U / kMinUnits));
    auto start = [&](long long c) { return c >= Ge ? U : (c * U) / Ge; };
    auto cta_of = [&](long long u) {
      long long c = (u * Ge) / U;
      while (c + 1 < Ge && start(c + 1) <= u) ++c;
      while (c > 0 && start(c) > u) --c;
      return c;
    };
    for (int c = 0; c < grid; ++c) {
      MkCtaPlan& pl = (*plan)[static_cast<std::size_t>(c) * 5 + sh];
      const long long u0 = start(c), u1 = start(c + 1);
      for (long long u = u0; u < u1;) {
        if (pl.nseg >= kMkMaxSeg) return false;
        MkSeg s{};
        s.t = static_cast<int>(u / KT);
        s.k0 = static_cast<int>(u % KT);
        s.k1 = static_cast<int>(std::min<long long>(KT, s.k0 + (u1 - u)));
        s.slot_self = u == u0 ? 0 : 1;
        s.c_first = static_cast<int>(cta_of(s.t * KT));
        s.c_last = static_cast<int>(cta_of(s.t * KT + KT - 1));
        s.first_slot = start(s.c_first) < s.t * KT ? 1 : 0;
        pl.seg[pl.nseg++] = s;
        u += s.k1 - s.k0;
      }
    }
  }
  for (int xk = 4; xk <= kMkMaxKt; xk *= 2) {
    bool ok = true;
    for (MkCtaPlan& pl : *plan) {
      unsigned long long seen = 0;
      pl.nkt = 0;
      for (int i = 0; i < pl.nseg && ok; ++i)
        for (int kt = pl.seg[i].k0; kt < pl.seg[i].k1; ++kt) {
          const unsigned long long bit = 1ull << (kt % xk);
          if (seen & bit) {
            ok = false;  // a second segment revisits kt: allowed only if it is the same k-tile
            for (int j = 0; j < pl.nkt; ++j)
              if (pl.kt[j] == kt) ok = true;
            if (!ok) break;
            continue;
          }
          seen |= bit;
          pl.kt[pl.nkt++] = static_cast<short>(kt);
        }
      if (!ok) break;
    }
    if (!ok) continue;
    const int st = (kSmemBudget - kSmemFixed - xk * kTileX) / kTileW;
    if (st < 3) return false;
    *xs_kt = xk;
    *stages = st < kMaxStages ? st : kMaxStages;
    *smem_bytes = kSmemFixed + xk * kTileX + *stages * kTileW;
    return true;
  }
  return false;
}

void decode_mk(const MkParams& p, int grid, int smem_bytes, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(decode_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
    uniform_carveout(reinterpret_cast<const void*>(decode_mk_kernel));
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, decode_mk_kernel, p);
}

}  // namespace moa::k
