// Decode GEMV on the tensor cores ("swap AB"): for R <= 16 activation rows
//   D[128 weight rows][16] = W_tile[128][K] . X[16][K]^T     (tcgen05, TMEM)
// so the weight tile is the M = 128 operand and the few decode rows are
// N = 16: the tensor pipe does the dot products for free and the kernel is a
// pure HBM stream of weights.  Work item = (128-row weight tile, K split);
// weights and activations arrive by TMA (SWIZZLE_128B) through a 6-stage
// mbarrier ring, one elected thread issues tcgen05.mma, 4 warps read the
// 128 x 16 fp32 accumulator back with tcgen05.ld (thread = weight row, 16
// registers = activation rows).  With K split over S CTAs, each writes a
// partial tile and the last CTA to arrive sums the S partials in split order
// and runs the epilogue (deterministic; S depends on (N, K) only).
// Epilogues: the GEMV path's (RoPE + KV append, residual, SwiGLU, fp32);
// RoPE / gate-up partners are adjacent weight rows = adjacent lanes.
#include <cstdio>
#include <cstdlib>
#include <set>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "stamp.cuh"

namespace moa::k {

namespace {

using namespace tc;

// 5-stage ring: 92 KB, two CTAs per SM (measured against 3 / 4 stages: the
// 8B decode tick is 8% / 2% slower with them)
constexpr int kM = 128, kN = 16, kBK = 64, kStages = 5;
constexpr int kTileW = kM * kBK * 2;  // 16 KB
constexpr int kTileX = kN * kBK * 2;  // 2 KB
constexpr int kSmem = kStages * (kTileW + kTileX) + 1024 + 256;
constexpr std::uint32_t kIdesc = idesc_bf16(kM, kN);
// Wide variants for ticks of 17..32 / 33..64 rows (incremental-prefill
// chunks): the same weight stream against a 32- / 64-row activation tile (MMA
// N = 32 / 64), a 4- / 3-stage ring so two CTAs still fit an SM next to the
// 16 / 32 KB split-K landing buffer.
template <int NC>
struct GvCfg {
  static constexpr int stages = NC == 16 ? kStages : NC == 32 ? 4 : 3;
  static constexpr int tmem_cols = NC < 32 ? 32 : NC;
  static constexpr int tile_x = NC * kBK * 2;
  static constexpr int smem = stages * (kTileW + tile_x) + 1024 + 256;
  static constexpr std::uint32_t idesc = idesc_bf16(kM, NC);
};

// Operands of the epilogue that do not depend on the MMA, loaded while the
// weights stream: the residual rows x[r][n] (final once the previous kernel
// completed), and for the QKV epilogue the rows' descriptors and RoPE factors
// (tick metadata / static tables).  Only rows r < R are touched.
struct EpiPre {
  float res[16];
  float2 cs[16];
  int kv[16], pos[16];
};

// The loads are pinned here (an empty asm consumes each value): without it the
// compiler sinks them to their use in the epilogue, putting the L2 round
// trips back on the critical path (measured: 2.4 us of RoPE epilogue per 8B
// QKV launch).
template <int EPI, int NR>
__device__ __forceinline__ void epi_preload(const GemvArgs& a, int n, int R, EpiPre& p, int rb = 0) {
  // rows rb .. rb + NR - 1 (NR <= 16) of the tick; predicated loads (no early
  // exit), so every row's load is in flight at once: one L2 round trip per
  // chunk instead of one (two for the QKV RoPE factors) per row -- the wide
  // variants run this on their critical path for the rows past the first 16
  if (EPI == kEpiResidual) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
      p.res[r] = (rb + r < R && n < a.N) ? __ldcg(a.out + static_cast<long long>(rb + r) * a.N + n) : 0.f;
#pragma unroll
    for (int r = 0; r < NR; ++r) asm volatile("" ::"f"(p.res[r]));
  } else if (EPI == kEpiQkv) {
    const int hd = a.hd, half = hd / 2, qk_cols = (a.nh + a.nkv) * hd;
    const int e = (n % hd) / 2;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int2 kp = rb + r < R ? *reinterpret_cast<const int2*>(a.rows + rb + r) : make_int2(0, 0);
      p.kv[r] = kp.x;
      p.pos[r] = kp.y;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r)
      p.cs[r] = (rb + r < R && n < qk_cols) ? __ldg(a.rope + static_cast<long long>(p.pos[r]) * half + e)
                                             : make_float2(1.f, 0.f);
#pragma unroll
    for (int r = 0; r < NR; ++r) asm volatile("" ::"f"(p.cs[r].x), "f"(p.cs[r].y), "r"(p.kv[r]), "r"(p.pos[r]));
  }
}

template <int EPI, int NR>
__device__ __forceinline__ void epilogue(const GemvArgs& a, int n, int R, const float (&v)[16], const EpiPre& pre, int rb = 0) {
  // v[r], pre.*[r]: row rb + r of the tick
  const int lane = threadIdx.x & 31;
  if (EPI == kEpiResidual && a.ssq_out) {
    // residual + per-16-column sums of squares of the new rows (the next
    // RMSNorm's statistics; 16 consecutive lanes = 16 consecutive columns)
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (rb + r >= R) break;
      float nv = 0.f;
      if (n < a.N) {
        nv = pre.res[r] + v[r];
        a.out[static_cast<long long>(rb + r) * a.N + n] = nv;
        if (a.xb_out) a.xb_out[static_cast<long long>(rb + r) * a.N + n] = __float2bfloat16_rn(nv);  // next GEMV's operand
      }
      float sq = nv * nv;
      sq += __shfl_xor_sync(0xffffffffu, sq, 1);
      sq += __shfl_xor_sync(0xffffffffu, sq, 2);
      sq += __shfl_xor_sync(0xffffffffu, sq, 4);
      sq += __shfl_xor_sync(0xffffffffu, sq, 8);
      if ((lane & 15) == 0 && n < a.N) a.ssq_out[static_cast<long long>(rb + r) * (a.N / 16) + n / 16] = sq;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    if (rb + r >= R) break;  // R is CTA-uniform
    const float x = v[r];
    const float partner = __shfl_xor_sync(0xffffffffu, x, 1);  // weight row n ^ 1
    if (n >= a.N) continue;
    switch (EPI) {
      case kEpiF32:
        a.out[static_cast<long long>(rb + r) * a.N + n] = x;
        break;
      case kEpiResidual:
        a.out[static_cast<long long>(rb + r) * a.N + n] = pre.res[r] + x;
        break;
      case kEpiSwiGlu:
        if (!(n & 1))
          a.out_bf16[static_cast<long long>(rb + r) * (a.N / 2) + n / 2] = __float2bfloat16_rn(x / (1.0f + __expf(-x)) * partner);
        break;
      case kEpiQkv: {
        const RowDesc rd{pre.kv[r], pre.pos[r], 0, 0};
        const int hd = a.hd, half = hd / 2, qk_cols = (a.nh + a.nkv) * hd;
        if (n < qk_cols) {
          if (n & 1) break;
          const int head = n / hd, e = (n % hd) / 2;
          const float2 cs = pre.cs[r];
          const float y0 = __fsub_rn(__fmul_rn(x, cs.x), __fmul_rn(partner, cs.y));
          const float y1 = __fadd_rn(__fmul_rn(partner, cs.x), __fmul_rn(x, cs.y));
          bf16* dst = head < a.nh ? a.out_bf16 + (static_cast<long long>(rb + r) * a.nh + head) * hd
                                  : a.kpool + rd.kv * a.kv_stride + a.layer_off +
                                        (static_cast<long long>(head - a.nh) * a.max_ctx + rd.pos) * hd;
          dst[e] = __float2bfloat16_rn(y0);
          dst[e + half] = __float2bfloat16_rn(y1);
        } else {
          const int vc = n - qk_cols, kh = vc / hd, e = vc % hd;
          a.vpool[rd.kv * a.kv_stride + a.layer_off + (static_cast<long long>(kh) * a.max_ctx + rd.pos) * hd + e] =
              __float2bfloat16_rn(x);
        }
        break;
      }
    }
  }
}

__device__ __forceinline__ std::uint32_t dsmem_addr(std::uint32_t local, int rank) {
  std::uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
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

// LM head epilogue: per logits row, greedy statistics over this tile's 128
// vocab entries (warp then CTA merge, fixed order), then the last CTA merges
// all tiles and writes token / logprob / entropy.
__device__ void lm_stats_epilogue(const GemvArgs& a, int n, int R, const float (&v)[16], int tile, int ntiles) {
  __shared__ LmStat sm[4][kN];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const LmStat none{-INFINITY, 0.f, 0.f, 0x7fffffff};
#pragma unroll
  for (int r = 0; r < kN; ++r) {
    if (r >= R) break;  // R is CTA-uniform: no work (and no shuffles) for absent rows
    const bool ok = n < a.N;
    if (ok && a.logits) a.logits[static_cast<long long>(r) * a.N + n] = v[r];
    LmStat st = ok ? LmStat{v[r], 1.f, 0.f, n} : none;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const LmStat o = shfl_stat(st, off);
      st = (lane & off) ? stat_merge(o, st) : stat_merge(st, o);
    }
    if (lane == 0) sm[warp][r] = st;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    LmStat st = sm[0][threadIdx.x];
    for (int w = 1; w < 4; ++w) st = stat_merge(st, sm[w][threadIdx.x]);
    a.lm_part[static_cast<long long>(threadIdx.x) * ntiles + tile] = st;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.lm_cnt, 1) == ntiles - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int r = warp; r < R; r += 4) {
    LmStat st = none;
    const float4* pr = reinterpret_cast<const float4*>(a.lm_part + static_cast<long long>(r) * ntiles);
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
      const int oi = a.out_idx[r];
      const float ls = logf(st.s);
      a.out_tok[oi] = st.idx;
      a.out_lp[oi] = -ls;
      a.out_ent[oi] = ls - st.t / st.s;
    }
  }
  if (threadIdx.x == 0) *a.lm_cnt = 0;
}

template <int EPI, int NR, int NC>
__global__ void __launch_bounds__(128)
gemv_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, const GemvArgs a,
               int S, float* __restrict__ ws, int* __restrict__ cnt) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  // Normed GEMVs (RMSNorm on the fp32 product, oracle/model.py normed_linear):
  // X = bf16(x) arrives by TMA like any activation; the rows' inverse RMS come
  // from the producers' 16-column sums of squares (a.ssq) or a prep kernel
  // (a.inv), computed while the weights stream and applied in the epilogue.
  const bool scaled = a.ssq != nullptr || a.inv != nullptr;
  using G = GvCfg<NC>;
  constexpr int stages = G::stages, kTileX = G::tile_x;
  unsigned char* sw = smem;
  unsigned char* sx = smem + stages * kTileW;  // per-stage X tiles
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(sx + stages * kTileX);
  std::uint64_t* empty = full + stages;
  std::uint64_t* done = empty + kStages;
  std::uint64_t* inv_bar = done + 1;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(inv_bar + 1);
  __shared__ float inv_s[NC];
  __shared__ float inv_red[2][NC];
  // split-K landing buffer: [src rank][row of this CTA's 128/S slice][NC] fp32
  __shared__ __align__(16) float land[kM * NC];
  __shared__ __align__(8) std::uint64_t land_bar;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int m0 = tile * kM;
  const int KT = a.K / kBK, kt0 = split * KT / S, kt_n = (split + 1) * KT / S - kt0;
  const std::uint32_t wtx = kTileW + kTileX;

  if (threadIdx.x == 0) {
    prefetch_tmap(&map_w);
    prefetch_tmap(&map_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_init(inv_bar, 1);
    if (S > 1) {
      mbar_init(&land_bar, 1);
      mbar_expect_tx(&land_bar, kM * NC * 4);  // every rank's slice of this CTA's rows (128/S x 16 x S)
    }
    mbar_fence_init();
  }
  __shared__ unsigned long long cst[kChainPhases];
  const unsigned stag = (5u << 16) | (static_cast<unsigned>(EPI) << 12) | ((a.K >> 4) & 0xfff);
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  const int R = a.meta ? __ldcg(a.meta) : a.R;  // tick metadata: not produced by the previous kernel
  // Dependents may launch now: they prefetch their own weights while this
  // grid runs, then wait (griddepcontrol.wait) for its completion before
  // reading its outputs.  Grids are sized to one CTA per SM, so this grid and
  // the next fit side by side.
  pdl_launch_dependents();
  if (warp == 0) tmem_alloc<G::tmem_cols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  // split-K: announce this CTA's landing barrier as initialised (waited on
  // just before the partials are pushed, long after)
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");

  // Weight tiles do not depend on the previous kernel: the first ring's worth
  // is issued before waiting on it (PDL).
  int kt_issued = 0;
  const std::uint64_t wpol = a.evict_first ? policy_evict_first() : 0;
  auto load_w = [&](int stage, int kt) {
    if (a.evict_first)
      tma_load_2d_hint(sw + stage * kTileW, &map_w, &full[stage], (kt0 + kt) * kBK, m0, wpol);
    else
      tma_load_2d(sw + stage * kTileW, &map_w, &full[stage], (kt0 + kt) * kBK, m0);
  };
  if (warp == 0 && lane == 0) {
    for (; kt_issued < kt_n && kt_issued < stages; ++kt_issued) {
      mbar_expect_tx(&full[kt_issued], wtx);
      load_w(kt_issued, kt_issued);
    }
  }
  if (warp == 0 && lane == 0) {
    // TMA producer (the rest of the weight stream; activations after the PDL wait)
    int kt = kt_issued;
    pdl_wait();
    for (int j = 0; j < kt; ++j) tma_load_2d(sx + j * kTileX, &map_x, &full[j], (kt0 + j) * kBK, 0);
    for (; kt < kt_n; ++kt) {
      const int s = kt % stages;
      mbar_wait(&empty[s], ((kt / stages) - 1) & 1);
      mbar_expect_tx(&full[s], wtx);
      load_w(s, kt);
      tma_load_2d(sx + s * kTileX, &map_x, &full[s], (kt0 + kt) * kBK, 0);
    }

  } else if (warp == 1 && lane == 0) {
    for (int kt = 0; kt < kt_n; ++kt) {
      const int s = kt % stages;
      mbar_wait(&full[s], (kt / stages) & 1);
      if (kt == 0) chain_mark(cst, 4);
      tc_fence_after();
      const std::uint32_t w0 = smem_u32(sw + s * kTileW), x0 = smem_u32(sx + s * kTileX);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) umma_bf16(tmem, umma_desc(w0 + k * 32), umma_desc(x0 + k * 32), G::idesc, (kt | k) ? 1u : 0u);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();
  pdl_wait();  // every epilogue thread reads the previous kernel's outputs (rows, residual)
  if (threadIdx.x == 64) chain_mark(cst, 1);
  // this thread's epilogue row: its TMEM lane, or with split-K its reduced row
  const int row = warp * 32 + lane;
  const int per = kM / S;
  const int n_epi = S == 1 ? m0 + row : (row < per ? m0 + split * per + row : a.N);
  EpiPre pre;
  if (EPI != kEpiLmStats) epi_preload<EPI, NR < 16 ? NR : 16>(a, n_epi, R, pre);
  if (scaled && warp >= 2) {
    // warps 2-3 (idle while the weights stream): each live row's inverse RMS,
    // from the producers' sums of squares (one float4 per thread per row, in a
    // fixed order) or from the prep kernel's values
    const int t = threadIdx.x - 64;
    if (a.ssq) {
      const int g4 = a.K / 64;  // float4 groups of 16-column partials per row (K <= 4096: <= 64)
#pragma unroll
      for (int r0 = 0; r0 < NR; r0 += 16) {  // batches of <= 16 rows: all loads of a batch in flight
        constexpr int NB = NR < 16 ? NR : 16;
        float4 b[NB];
#pragma unroll
        for (int r = 0; r < NB; ++r)
          b[r] = (r0 + r < R && t < g4)
                     ? __ldcg(reinterpret_cast<const float4*>(a.ssq + static_cast<long long>(r0 + r) * (a.K / 16)) + t)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < NB; ++r) {
          if (r0 + r >= R) break;
          float v = (b[r].x + b[r].y) + (b[r].z + b[r].w);
#pragma unroll
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) inv_red[warp - 2][r0 + r] = v;
        }
      }
      asm volatile("bar.sync 2, 64;" ::: "memory");
      if (t < NC) inv_s[t] = t < R ? 1.0f / sqrtf((inv_red[0][t] + inv_red[1][t]) / static_cast<float>(a.K) + a.eps) : 0.f;
    } else if (t < NC) {
      inv_s[t] = t < R ? __ldcg(a.inv + t) : 0.f;
    }
    asm volatile("bar.sync 2, 64;" ::: "memory");
    if (t == 0) mbar_arrive(inv_bar);
  }
  mbar_wait(done, 0);
  tc_fence_after();
  if (threadIdx.x == 64) chain_mark(cst, 3);

  const int n = m0 + row;
  constexpr int NH = NC / 16;  // 16-column halves of the accumulator
  float v[NH][16];
#pragma unroll
  for (int h = 0; h < NH; ++h) tmem_ld16(tmem + (static_cast<std::uint32_t>(warp * 32) << 16) + 16 * h, v[h]);
  if (scaled) mbar_wait(inv_bar, 0);
  auto scale_rows = [&](float (&u)[16], int rb) {
    if (!scaled) return;
#pragma unroll
    for (int r = 0; r < 16; ++r) u[r] *= inv_s[rb + r];
  };
  // Wide variants: the 16-row chunks in a rolled loop, the epilogue operands
  // of rows past the first 16 loaded per chunk (the first 16 rows' were
  // preloaded while the weights streamed).  Unrolled, the 64-row QKV epilogue
  // was ~20k instructions run once from a cold instruction cache (ncu: 57% of
  // the warps' samples at the final barrier waiting on it, 76 us per 8B launch).
  auto run_epilogue = [&](int n_row) {
    if constexpr (NH == 1) {
      scale_rows(v[0], 0);
      epilogue<EPI, NR < 16 ? NR : 16>(a, n_row, R, v[0], pre, 0);
    } else {
      // one copy of the 16-row epilogue, cold once, then warm
#pragma unroll 1
      for (int h = 0; h < NH; ++h) {
        if (16 * h >= R) break;
        float u[16];
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
          if (hh == h)
#pragma unroll
            for (int r = 0; r < 16; ++r) u[r] = v[hh][r];
        scale_rows(u, 16 * h);
        EpiPre p1 = pre;
        if (h > 0) epi_preload<EPI, 16>(a, n_row, R, p1, 16 * h);
        epilogue<EPI, 16>(a, n_row, R, u, p1, 16 * h);
      }
    }
  };
  if constexpr (EPI == kEpiLmStats) {
    static_assert(NC == 16, "LM statistics: 16 rows");
    scale_rows(v[0], 0);
    lm_stats_epilogue(a, n, R, v[0], tile, gridDim.x);  // S == 1 for the LM head
  } else {
    // one call site of the (inlined) epilogue: run by every thread (S == 1) or
    // by the warps holding reduced rows (split-K)
    int n_run = n;
    bool run = true;
    if (S > 1) {
      // Split-K inside a thread-block cluster (the S CTAs of this weight tile):
      // CTA q reduces weight rows [q*128/S, (q+1)*128/S).  Every CTA pushes the
      // partial rows owned by q straight into q's landing buffer with st.async
      // (DSMEM stores that complete transactions on q's mbarrier), so a reducer
      // waits only for its own data -- no cluster-wide barrier, no remote loads
      // -- then sums the S partials in rank order (deterministic) and runs the
      // epilogue of its rows.
      const int q = row / per, rq = row % per;
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every landing barrier is initialised
      {
        const std::uint32_t dst = dsmem_addr(smem_u32(land + (split * per + rq) * NC), q);
        const std::uint32_t bar = dsmem_addr(smem_u32(&land_bar), q);
  #pragma unroll
        for (int h = 0; h < NH; ++h)
  #pragma unroll
          for (int i = 0; i < 4; ++i)
            asm volatile(
                "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                    dst + 64 * h + 16 * i),
                "f"(v[h][4 * i]), "f"(v[h][4 * i + 1]), "f"(v[h][4 * i + 2]), "f"(v[h][4 * i + 3]), "r"(bar)
                : "memory");
      }
      if (threadIdx.x == 0) chain_mark(cst, 5);
      if constexpr (NH > 1) {
        // Wide variants: the reduced rows' epilogues are spread over all four
        // warps as units of (32 reduced rows, one 16-column chunk): with one
        // warp per CTA holding reduced rows, the 64-row QKV epilogue ran ~5.7k
        // dependent instructions on a single warp (ncu: the other warps' samples
        // at the final barrier, 57% of the kernel).  Same split order, same sums.
        mbar_wait(&land_bar, 0);
        const int units = (per + 31) / 32 * NH;
  #pragma unroll 1
        for (int un = warp; un < units; un += 4) {
          const int h = un % NH, rr = un / NH * 32 + lane;
          if (16 * h >= R) continue;  // warp-uniform
          const bool mine = rr < per;
          float u[16];
  #pragma unroll
          for (int i = 0; i < 16; ++i) u[i] = 0.f;
          if (mine)
            for (int src = 0; src < S; ++src) {
              const float4* p = reinterpret_cast<const float4*>(land + (src * per + rr) * NC + 16 * h);
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 t = p[i];
                u[4 * i] += t.x;
                u[4 * i + 1] += t.y;
                u[4 * i + 2] += t.z;
                u[4 * i + 3] += t.w;
              }
            }
          const int nn = mine ? m0 + split * per + rr : a.N;
          scale_rows(u, 16 * h);
          EpiPre p1;
          epi_preload<EPI, 16>(a, nn, R, p1, 16 * h);
          epilogue<EPI, 16>(a, nn, R, u, p1, 16 * h);
        }
        run = false;
      } else if (warp * 32 < per) {  // warps holding at least one reduced row (whole warps: the epilogue shuffles)
        mbar_wait(&land_bar, 0);
        const bool mine = row < per;
        const int wr = split * per + (mine ? row : 0);
  #pragma unroll
        for (int h = 0; h < NH; ++h)
  #pragma unroll
          for (int i = 0; i < 16; ++i) v[h][i] = 0.f;
        if (mine)
          for (int src = 0; src < S; ++src) {
            const float4* p = reinterpret_cast<const float4*>(land + (src * per + row) * NC);
  #pragma unroll
            for (int h = 0; h < NH; ++h)
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 t = p[4 * h + i];
                v[h][4 * i] += t.x;
                v[h][4 * i + 1] += t.y;
                v[h][4 * i + 2] += t.z;
                v[h][4 * i + 3] += t.w;
              }
          }
        if (threadIdx.x == 0) chain_mark(cst, 6);
        n_run = mine ? m0 + wr : a.N;
      } else {
        run = false;
      }
    }
    if (run) run_epilogue(n_run);
  }
  if (threadIdx.x == 0) chain_mark(cst, 7);  // this thread's epilogue done
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, stag);
  }
  if (warp == 0) tmem_dealloc<G::tmem_cols>(tmem);
}


// ---------------------------------------------------------------------------
// Persistent LM head (greedy statistics), one CTA per SM.  CTA c owns the
// contiguous vocab tiles [c*T/G, (c+1)*T/G); the weight ring runs across its
// tiles without a break and every tile accumulates into its own 16 TMEM
// columns (<= 32 tiles per CTA), so the MMAs never wait for an epilogue.  The
// epilogue warps fold each finished tile into a per-lane running statistic
// with single-column TMEM loads (tile order), reduce once per row across the
// warp and the four lane quarters, write one partial per row, and the last
// CTA merges the G partials in CTA order -> token / logprob / entropy.
constexpr int kLmStages = 8;       // weight+activation ring (activations by TMA)
constexpr int kLmMaxStages = 16;   // weight ring with the norm folded in
constexpr int kLmMaxTiles = 32;    // TMEM: 32 tiles x 16 columns
constexpr int kLmSmem = kLmStages * (kTileW + kTileX) + 1024 + 1024;
// norm-folded LM head: all K tiles of the normalised rows staged once + a weight ring
__host__ __device__ inline int lm_fold_stages(int K) {
  const int st = (220 * 1024 - (K / kBK) * kTileX) / kTileW;
  return st > kLmMaxStages ? kLmMaxStages : st;
}
inline int lm_fold_smem(int K) { return lm_fold_stages(K) * kTileW + (K / kBK) * kTileX + 1024 + 1024; }

__device__ __forceinline__ float tmem_ld1(std::uint32_t taddr) {
  std::uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return __uint_as_float(r);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int COLS>
__device__ __forceinline__ void lm_tmem_alloc(std::uint32_t* slot) { tmem_alloc<COLS>(slot); }

__global__ void __launch_bounds__(192, 1)
lm_head_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, const GemvArgs a,
                  LmStat* __restrict__ part, int* __restrict__ cnt) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  __shared__ unsigned long long cst[kChainPhases];
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  const bool fold = a.X != nullptr;  // normalise the selected residual rows in-kernel
  const int KT = a.K / kBK;
  const int stages = fold ? lm_fold_stages(a.K) : kLmStages;
  unsigned char* sw = smem;
  unsigned char* sx = smem + stages * kTileW;  // per-stage X tiles, or (fold) all KT normalised tiles
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(sx + (fold ? KT : kLmStages) * kTileX);
  std::uint64_t* empty = full + kLmMaxStages;
  std::uint64_t* accf = empty + kLmMaxStages;  // [kLmMaxTiles]: tile j accumulated
  std::uint64_t* xrdy = accf + kLmMaxTiles;    // fold: staging written
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(xrdy + 1);
  __shared__ LmStat red[4][kN];
  __shared__ bool last;
  __shared__ float inv_s[kN];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = (a.N + kM - 1) / kM, G = gridDim.x, c = blockIdx.x;
  const int t0 = static_cast<int>(static_cast<long long>(c) * T / G), t1 = static_cast<int>(static_cast<long long>(c + 1) * T / G);
  const int tmax = (T + G - 1) / G;  // tiles of the largest CTA (uniform TMEM allocation)
  const std::uint32_t wtx = fold ? kTileW : kTileW + kTileX;
  const LmStat none{-INFINITY, 0.f, 0.f, 0x7fffffff};

  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    prefetch_tmap(&map_w);
    if (!fold) prefetch_tmap(&map_x);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int j = 0; j < t1 - t0; ++j) mbar_init(&accf[j], 1);
    mbar_init(xrdy, 1);
    mbar_fence_init();
  }
  if (warp == 0) {
    if (tmax <= 2) lm_tmem_alloc<32>(tmem_slot);
    else if (tmax <= 4) lm_tmem_alloc<64>(tmem_slot);
    else if (tmax <= 8) lm_tmem_alloc<128>(tmem_slot);
    else if (tmax <= 16) lm_tmem_alloc<256>(tmem_slot);
    else lm_tmem_alloc<512>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: weights before the PDL wait, activations after
      const int total = (t1 - t0) * KT;
      const std::uint64_t wpol = a.evict_first ? policy_evict_first() : 0;
      auto load_w = [&](int stage, int qq) {
        if (a.evict_first)
          tma_load_2d_hint(sw + stage * kTileW, &map_w, &full[stage], (qq % KT) * kBK, (t0 + qq / KT) * kM, wpol);
        else
          tma_load_2d(sw + stage * kTileW, &map_w, &full[stage], (qq % KT) * kBK, (t0 + qq / KT) * kM);
      };
      int q = 0;
      for (; q < total && q < stages; ++q) {
        mbar_expect_tx(&full[q], wtx);
        load_w(q, q);
      }
      if (!fold) {
        pdl_wait();
        for (int j = 0; j < q; ++j) tma_load_2d(sx + j * kTileX, &map_x, &full[j], (j % KT) * kBK, 0);
      }
      for (; q < total; ++q) {
        const int s = q % stages;
        mbar_wait(&empty[s], ((q / stages) - 1) & 1);
        mbar_expect_tx(&full[s], wtx);
        load_w(s, q);
        if (!fold) tma_load_2d(sx + s * kTileX, &map_x, &full[s], (q % KT) * kBK, 0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: tile j -> TMEM columns [16j, 16j + 16)
      int q = 0;
      if (fold && t1 > t0) mbar_wait(xrdy, 0);  // the normalised rows are staged
      chain_mark(cst, 5);
      for (int t = t0; t < t1; ++t) {
        const int j = t - t0;
        tc_fence_after();
        for (int kt = 0; kt < KT; ++kt, ++q) {
          const int s = q % stages;
          mbar_wait(&full[s], (q / stages) & 1);
          tc_fence_after();
          const std::uint32_t w0 = smem_u32(sw + s * kTileW), x0 = smem_u32(sx + (fold ? kt : s) * kTileX);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(tmem + j * kN, umma_desc(w0 + k * 32), umma_desc(x0 + k * 32), kIdesc, (kt | k) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&accf[j]);
      }
      chain_mark(cst, 7);
    }
    __syncwarp();
  } else {
    // epilogue warps 2-5: TMEM lane quarter = warp % 4
    const int R = a.meta ? __ldcg(a.meta) : a.R;  // tick metadata, before the PDL wait
    pdl_wait();
    if (threadIdx.x == 64) chain_mark(cst, 1);
    if (fold) {
      // stage bf16(x[sel[r]]) for every k-tile (128B-swizzled K-major); the
      // rows' inverse RMS scale the logits (RMSNorm on the fp32 product).
      // With the producer's bf16 copy of x and its 16-column sums of squares
      // (a.A, a.ssq: decode ticks) both are plain loads; else from fp32 x.
      // Every thread issues all its loads of a batch before using them.
      const int et0 = threadIdx.x - 64;
      const bool xb = a.A != nullptr && a.ssq != nullptr;
      __shared__ int sel_s[kN];
      if (et0 < kN) sel_s[et0] = et0 < R ? __ldg(a.sel + et0) : 0;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      {
        const int r = et0 >> 3, j = et0 & 7;  // 8 threads per row
        float ss = 0.f;
        if (r < R) {
          if (xb) {  // K / 16 partials per row: K / 128 float4 per thread
            const float4* pr = reinterpret_cast<const float4*>(a.ssq + static_cast<long long>(sel_s[r]) * (a.K / 16));
            float4 b[8];
            for (int q0 = j; q0 < a.K / 64; q0 += 64) {
#pragma unroll
              for (int u = 0; u < 8; ++u) b[u] = q0 + 8 * u < a.K / 64 ? __ldcg(pr + q0 + 8 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int u = 0; u < 8; ++u) ss += (b[u].x + b[u].y) + (b[u].z + b[u].w);
            }
          } else {
            const float4* xr = reinterpret_cast<const float4*>(a.X + static_cast<long long>(sel_s[r]) * a.K);
            float4 b[8];
            for (int q0 = j; q0 < a.K / 4; q0 += 64) {
#pragma unroll
              for (int u = 0; u < 8; ++u) b[u] = q0 + 8 * u < a.K / 4 ? __ldg(xr + q0 + 8 * u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                ss = fmaf(b[u].x, b[u].x, ss);
                ss = fmaf(b[u].y, b[u].y, ss);
                ss = fmaf(b[u].z, b[u].z, ss);
                ss = fmaf(b[u].w, b[u].w, ss);
              }
            }
          }
        }
        ss += __shfl_xor_sync(0xffffffffu, ss, 1);
        ss += __shfl_xor_sync(0xffffffffu, ss, 2);
        ss += __shfl_xor_sync(0xffffffffu, ss, 4);
        if (j == 0 && r < kN) inv_s[r] = r < R ? 1.0f / sqrtf(ss / static_cast<float>(a.K) + a.eps) : 0.f;
      }
      const int nchunk = KT * R * 8;  // (k-tile, row, 16-byte chunk of 8 elements)
      for (int c0 = et0; c0 < nchunk; c0 += 128 * 8) {
        uint4 raw[8];
        float4 xa[8], xc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ch = c0 + 128 * u;
          if (ch >= nchunk) continue;
          const int t = ch / (R * 8), r = (ch >> 3) % R, cc = ch & 7;
          const long long off = static_cast<long long>(sel_s[r]) * a.K + t * kBK + cc * 8;
          if (xb) {
            raw[u] = __ldcg(reinterpret_cast<const uint4*>(a.A + off));
          } else {
            xa[u] = __ldg(reinterpret_cast<const float4*>(a.X + off));
            xc[u] = __ldg(reinterpret_cast<const float4*>(a.X + off + 4));
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int ch = c0 + 128 * u;
          if (ch >= nchunk) continue;
          const int t = ch / (R * 8), r = (ch >> 3) % R, cc = ch & 7;
          if (!xb) {
            __align__(16) bf16 o8[8];
            o8[0] = __float2bfloat16_rn(xa[u].x);
            o8[1] = __float2bfloat16_rn(xa[u].y);
            o8[2] = __float2bfloat16_rn(xa[u].z);
            o8[3] = __float2bfloat16_rn(xa[u].w);
            o8[4] = __float2bfloat16_rn(xc[u].x);
            o8[5] = __float2bfloat16_rn(xc[u].y);
            o8[6] = __float2bfloat16_rn(xc[u].z);
            o8[7] = __float2bfloat16_rn(xc[u].w);
            raw[u] = *reinterpret_cast<const uint4*>(o8);
          }
          *reinterpret_cast<uint4*>(sx + t * kTileX + r * 128 + ((cc ^ (r & 7)) * 16)) = raw[u];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et0 == 0) mbar_arrive(xrdy);
      if (et0 == 0) chain_mark(cst, 3);
    } else {
      // operand rows prepared by the prep kernel (bf16(x) by TMA), their inverse RMS in a.inv
      const int et0 = threadIdx.x - 64;
      if (et0 < kN) inv_s[et0] = et0 < R ? (a.inv ? __ldcg(a.inv + et0) : 1.f) : 0.f;
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    const int quarter = warp & 3;
    const int et = threadIdx.x - 64;  // 0..127
    const std::uint32_t tq = tmem + (static_cast<std::uint32_t>(quarter * 32) << 16);
    // one running statistic per (row, lane): rows outer, tiles inner
    // (single-column TMEM loads keep the code small for any row count)
    for (int j = 0; j < t1 - t0; ++j) mbar_wait(&accf[j], 0);
    tc_fence_after();
    if (et == 0) chain_mark(cst, 4);
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      LmStat st = none;
#pragma unroll 1
      for (int t = t0; t < t1; t += 4) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          v[u] = t + u < t1 ? tmem_ld1(tq + static_cast<std::uint32_t>((t + u - t0) * kN + r)) : 0.f;
        tmem_ld_wait();
        const float iv = inv_s[r];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] *= iv;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int n = (t + u) * kM + quarter * 32 + lane;
          if (t + u < t1 && n < a.N) {
            if (a.logits) a.logits[static_cast<long long>(r) * a.N + n] = v[u];
            st = stat_merge(st, LmStat{v[u], 1.f, 0.f, n});
          }
        }
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const LmStat o = shfl_stat(st, off);
        st = (lane & off) ? stat_merge(o, st) : stat_merge(st, o);
      }
      if (lane == 0) red[quarter][r] = st;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (et < R) {
      // quarters of one tile are vocab-ordered; across tiles the per-lane fold
      // already ran in tile order, so quarter order here is a fixed order
      LmStat st = red[0][et];
      for (int w = 1; w < 4; ++w) st = stat_merge(st, red[w][et]);
      __stcg(reinterpret_cast<float4*>(part + static_cast<long long>(et) * G + c),
             make_float4(st.m, st.s, st.t, __int_as_float(st.idx)));
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (et == 0) {
      unsigned prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt) : "memory");
      last = prev == static_cast<unsigned>(G - 1);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (last) {
      for (int r = et >> 5; r < R; r += 4) {
        LmStat st = none;
        const float4* pr = reinterpret_cast<const float4*>(part + static_cast<long long>(r) * G);
        for (int b0 = lane; b0 < G; b0 += 32 * 8) {
          float4 raw[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int bb = b0 + 32 * u;
            raw[u] = bb < G ? __ldcg(pr + bb) : make_float4(-INFINITY, 0.f, 0.f, __int_as_float(0x7fffffff));
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
          const int oi = a.out_idx[r];
          const float ls = logf(st.s);
          a.out_tok[oi] = st.idx;
          a.out_lp[oi] = -ls;
          a.out_ent[oi] = ls - st.t / st.s;
        }
      }
      if (et == 0) __stcg(cnt, 0);
      if (et == 0) chain_mark(cst, 6);
    }
    if (et == 0) {
      chain_mark(cst, 2);
      chain_flush(cst, 3u << 16);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    if (tmax <= 2) tmem_dealloc<32>(tmem);
    else if (tmax <= 4) tmem_dealloc<64>(tmem);
    else if (tmax <= 8) tmem_dealloc<128>(tmem);
    else if (tmax <= 16) tmem_dealloc<256>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

}  // namespace

void lm_head_tc(const TmaMap& map_w, const TmaMap& map_x, const GemvArgs& a, LmStat* part, int* cnt, int grid,
                cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lm_head_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 222 * 1024);
    uniform_carveout(reinterpret_cast<const void*>(lm_head_tc_kernel));
    attr = true;
  }
  const int T = (a.N + kM - 1) / kM;
  const int G = grid < T ? grid : T;
  if ((T + G - 1) / G > kLmMaxTiles) {
    std::fprintf(stderr, "lm_head_tc: %d vocab tiles over %d CTAs exceed %d tiles per CTA\n", T, G, kLmMaxTiles);
    std::abort();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = a.X ? lm_fold_smem(a.K) : kLmSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, lm_head_tc_kernel, *reinterpret_cast<const CUtensorMap*>(&map_w),
                     *reinterpret_cast<const CUtensorMap*>(&map_x), a, part, cnt);
}

MOA_CHAIN_STAMP_SETTER(gemv_tc_chain_stamp)

// K splits per weight tile: as many as keep the grid within one CTA per SM
// (148), at least 4 k-tiles per split (uneven splits allowed; the partials
// are summed in split order, so the result depends only on (N, K)).
int gemv_tc_splits(int N, int K, int epi) {
  const int tiles = (N + kM - 1) / kM, kts = K / kBK;
  if (epi == kEpiLmStats) return 1;
  static const int max_ctas = [] {  // MOA_GEMV_MAX_CTAS (A/B): cap on tiles x splits
    const char* e = std::getenv("MOA_GEMV_MAX_CTAS");
    return e ? std::atoi(e) : 2 * 148;
  }();
  int S = 1;  // power of two <= 8 (one cluster per tile), >= 4 k-tiles per split, <= 2 CTAs per SM
  while (S < 8 && tiles * S * 2 <= max_ctas && kts / (S * 2) >= 4) S *= 2;
  return S;
}

long long gemv_tc_ws_floats(int N, int K) {
  return static_cast<long long>((N + kM - 1) / kM) * gemv_tc_splits(N, K, kEpiF32) * kM * kN;
}

bool gemv_tc_norm_supported(const GemvArgs& a) {
  // inverse RMS from 16-column partials: one float4 of them per thread of two warps
  return gemv_tc_supported(a) && a.K % 64 == 0 && a.K <= 64 * 64;
}

bool gemv_tc_supported(const GemvArgs& a) {
  return a.R <= kGemvTcWideRows && (a.R <= kN || a.epi != kEpiLmStats) && a.K % kBK == 0 && a.N % 2 == 0 &&
         static_cast<long long>(a.N) * a.K >= (2LL << 20);
}

// One kernel per (epilogue, row bucket): the epilogue and its per-row loops
// are compiled for the bucket's row count only, so each launch runs a small,
// branch-free instruction stream (the generic kernel's qkv epilogue took
// ~1.3 us longer than the residual one at the same work, in every launch).
template <int EPI>
static void (*gemv_tc_pick(int R))(CUtensorMap, CUtensorMap, GemvArgs, int, float*, int*) {
  if (R <= 4) return gemv_tc_kernel<EPI, 4, 16>;
  if (R <= 8) return gemv_tc_kernel<EPI, 8, 16>;
  if (R <= 16 || EPI == kEpiLmStats) return gemv_tc_kernel<EPI, 16, 16>;
  if constexpr (EPI != kEpiLmStats) {
    if (R <= kGemvTcMidRows) return gemv_tc_kernel<EPI, 32, 32>;
    return gemv_tc_kernel<EPI, 64, 64>;
  }
  return nullptr;
}

void gemv_tc(const TmaMap& map_w, const TmaMap& map_x, const GemvArgs& a, float* ws, int* cnt, cudaStream_t st) {
  void (*kern)(CUtensorMap, CUtensorMap, GemvArgs, int, float*, int*) = nullptr;
  switch (a.epi) {
    case kEpiF32: kern = gemv_tc_pick<kEpiF32>(a.R); break;
    case kEpiResidual: kern = gemv_tc_pick<kEpiResidual>(a.R); break;
    case kEpiSwiGlu: kern = gemv_tc_pick<kEpiSwiGlu>(a.R); break;
    case kEpiQkv: kern = gemv_tc_pick<kEpiQkv>(a.R); break;
    default: kern = gemv_tc_pick<kEpiLmStats>(a.R); break;
  }
  const int box = gemv_tc_box_rows(a.R);
  const int smem = box == 16 ? GvCfg<16>::smem : box == 32 ? GvCfg<32>::smem : GvCfg<64>::smem;
  static std::set<const void*> attr;
  if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uniform_carveout(reinterpret_cast<const void*>(kern));
  }
  const int S = gemv_tc_splits(a.N, a.K, a.epi);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((a.N + kM - 1) / kM, S);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  if (pdl_enabled()) {
    attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (S > 1) {  // the S K-splits of a weight tile form one cluster (DSMEM reduction)
    attrs[na].id = cudaLaunchAttributeClusterDimension;
    attrs[na].val.clusterDim.x = 1;
    attrs[na].val.clusterDim.y = S;
    attrs[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(&map_w),
                     *reinterpret_cast<const CUtensorMap*>(&map_x), a, S, ws, cnt);
}

}  // namespace moa::k
