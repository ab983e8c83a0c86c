// Prefill GEMM on the 5th-generation tensor cores (sm_100a):
//   Y[M][N] = A[M][K] . W[N][K]^T, bf16 operands, fp32 accumulation in TMEM.
//
// Two kernels, one epilogue (RoPE + KV append / residual add / SwiGLU / fp32,
// normed maps scaled by the rows' inverse RMS):
//  * gemm_tc_kernel -- one CTA per 128 x 128 output tile, 4 warps (warp 0:
//    TMA producer, warp 1: MMA issuer, all four: epilogue), 3-stage ring, two
//    CTAs per SM so one's epilogue overlaps the other's main loop.  Used for
//    the chunked-prefill ticks (M <= 512 rows): N / 128 CTAs stream the
//    weights.
//  * gemm_tc_persistent_kernel -- prompt-prefill ticks (M > 512): one CTA per
//    SM loops over 128 x 256 tiles (M-fastest order: concurrent CTAs share a
//    weight tile in L2); warp 0 streams A and W k-tiles through a 3-stage
//    ring, warp 1 issues tcgen05.mma (M 128, N 256) into one of two TMEM
//    accumulators (2 x 256 columns), warps 2-5 run the epilogue of tile i
//    while the tensor core computes tile i + 1.
// With N along TMEM columns each thread holds consecutive columns of its row,
// so RoPE pairs and gate/up pairs (adjacent device columns) sit in one thread.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "stamp.cuh"

namespace moa::k {

namespace {

using namespace tc;

constexpr int kBM = 128, kBN = 128, kBK = 64, kStages = 3;
constexpr int kTileA = kBM * kBK * 2;  // 16 KB
constexpr int kTileB = kBN * kBK * 2;  // 16 KB
constexpr int kSmem = kStages * (kTileA + kTileB) + 1024 /*align*/ + 256 /*barriers*/;
constexpr std::uint32_t kIdesc = idesc_bf16(kBM, kBN);

// persistent kernel: 128 x 256 tiles, 3 stages (+ a 32 KB epilogue staging tile), 2 TMEM accumulators
constexpr int kPN = 256, kPStages = 3;
constexpr int kPTileB = kPN * kBK * 2;  // 32 KB
constexpr int kPStage = kTileA + kPTileB;
constexpr int kPStaging = kBM * kBN * 2;  // 32 KB: a 128 x 128 bf16 half-tile (QKV epilogue)
constexpr int kPSmem = kPStages * kPStage + kPStaging + 1024 + 256;
constexpr std::uint32_t kPIdesc = idesc_bf16(kBM, kPN);
constexpr int kPMinRows = 512;  // rows above which the persistent kernel runs

// Epilogue of one 128-row x 128-column block of the output: `tc` = TMEM
// address of this thread's lane and the block's first column, (row, n0) the
// output coordinates, `et` the thread's index among the 128 epilogue threads
// and `sync` a barrier over them; `st` is 32 KB of staging smem (QKV).
template <typename Sync>
__device__ __forceinline__ void block_epilogue(const GemvArgs& a, std::uint32_t tc, int row, bool row_ok, int live,
                                               int m0, int n0, int et, const RowDesc& rd, float rs, bf16* st,
                                               RowDesc* rds, Sync sync) {
  auto ld_scaled = [&](int c0, float (&v)[16]) {
    tmem_ld16(tc + static_cast<std::uint32_t>(c0), v);
    if (a.inv) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] *= rs;
    }
  };
  const int lr = row - m0;  // block-local row
  if (a.epi == kEpiQkv && kBN % a.hd == 0) {
    // RoPE + q / K / V rows staged as a bf16 tile in smem in natural head
    // order, then written out in 16-byte chunks: one head row (hd x 2 bytes)
    // per destination, instead of one 2-byte store per element scattered over
    // q and the KV pool (16-byte chunks XOR-ed with row % 16: a warp's threads
    // are 32 rows writing the same column)
    auto sti = [](int rr, int cc) { return rr * kBN + ((((cc >> 3) ^ (rr & 15))) << 3) + (cc & 7); };
    rds[lr] = rd;
    const int hd = a.hd, half = hd / 2, qk_cols = (a.nh + a.nkv) * hd;
    for (int c0 = 0; c0 < kBN; c0 += 16) {
      float v[16];
      __syncwarp();  // tcgen05.ld is warp-collective
      ld_scaled(c0, v);
      if (!row_ok) continue;
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const int n = n0 + c0 + i, cl = c0 + i;
        if (n < qk_cols) {
          const int e = (n % hd) / 2, hb = cl - (n % hd);  // tile-local head start
          const float2 cs = a.rope[static_cast<long long>(rd.pos) * half + e];
          const float x0 = v[i], x1 = v[i + 1];
          st[sti(lr, hb + e)] = __float2bfloat16_rn(__fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y)));
          st[sti(lr, hb + e + half)] = __float2bfloat16_rn(__fadd_rn(__fmul_rn(x1, cs.x), __fmul_rn(x0, cs.y)));
        } else {
          st[sti(lr, cl)] = __float2bfloat16_rn(v[i]);
          st[sti(lr, cl + 1)] = __float2bfloat16_rn(v[i + 1]);
        }
      }
    }
    sync();
    const int cpr = kBN / 8;  // 16-byte chunks per tile row
    for (int c = et; c < kBM * cpr; c += 128) {
      const int rl = c / cpr, ch = c % cpr, r = m0 + rl;
      const int n = n0 + ch * 8;
      if (r >= live || n >= a.N) continue;
      const RowDesc d = rds[rl];
      const uint4 val = *reinterpret_cast<const uint4*>(st + sti(rl, ch * 8));
      const int head = n / hd, e = n % hd;
      bf16* dst;
      if (head < a.nh)
        dst = a.out_bf16 + (static_cast<long long>(r) * a.nh + head) * hd + e;
      else if (head < a.nh + a.nkv)
        dst = a.kpool + d.kv * a.kv_stride + a.layer_off + (static_cast<long long>(head - a.nh) * a.max_ctx + d.pos) * hd + e;
      else
        dst = a.vpool + d.kv * a.kv_stride + a.layer_off +
              (static_cast<long long>(head - a.nh - a.nkv) * a.max_ctx + d.pos) * hd + e;
      *reinterpret_cast<uint4*>(dst) = val;
    }
    sync();  // staging and rds are reused by the next block
    return;
  }
  for (int c0 = 0; c0 < kBN; c0 += 16) {
    float v[16];
    __syncwarp();  // tcgen05.ld is warp-collective
    ld_scaled(c0, v);
    if (!row_ok) continue;
    const int nb = n0 + c0;
    if (nb >= a.N) break;
    switch (a.epi) {
      case kEpiF32: {
        float4* o = reinterpret_cast<float4*>(a.out + static_cast<long long>(row) * a.N + nb);
#pragma unroll
        for (int i = 0; i < 4; ++i) o[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        break;
      }
      case kEpiResidual: {
        float4* o = reinterpret_cast<float4*>(a.out + static_cast<long long>(row) * a.N + nb);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float4 x = o[i];
          x.x += v[4 * i];
          x.y += v[4 * i + 1];
          x.z += v[4 * i + 2];
          x.w += v[4 * i + 3];
          o[i] = x;
        }
        break;
      }
      case kEpiSwiGlu: {  // 8 outputs = one 16-byte store
        __align__(16) bf16 o8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float g = v[2 * i], u = v[2 * i + 1];
          o8[i] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
        }
        *reinterpret_cast<uint4*>(a.out_bf16 + static_cast<long long>(row) * (a.N / 2) + nb / 2) =
            *reinterpret_cast<const uint4*>(o8);
        break;
      }
      case kEpiQkv: {  // head dim not dividing the block: per-element RoPE stores
        const int hd = a.hd, half = hd / 2;
        const int qk_cols = (a.nh + a.nkv) * hd;
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const int n = nb + i;
          if (n < qk_cols) {
            const int head = n / hd, e = (n % hd) / 2;
            const float2 cs = a.rope[static_cast<long long>(rd.pos) * half + e];
            const float x0 = v[i], x1 = v[i + 1];
            const float y0 = __fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y));
            const float y1 = __fadd_rn(__fmul_rn(x1, cs.x), __fmul_rn(x0, cs.y));
            bf16* dst = head < a.nh ? a.out_bf16 + (static_cast<long long>(row) * a.nh + head) * hd
                                    : a.kpool + rd.kv * a.kv_stride + a.layer_off +
                                          (static_cast<long long>(head - a.nh) * a.max_ctx + rd.pos) * hd;
            dst[e] = __float2bfloat16_rn(y0);
            dst[e + half] = __float2bfloat16_rn(y1);
          } else {
            const int vc = n - qk_cols, kh = vc / hd, e = vc % hd;
            bf16* dst = a.vpool + rd.kv * a.kv_stride + a.layer_off +
                        (static_cast<long long>(kh) * a.max_ctx + rd.pos) * hd + e;
            dst[0] = __float2bfloat16_rn(v[i]);
            dst[1] = __float2bfloat16_rn(v[i + 1]);
          }
        }
        break;
      }
    }
  }
}

__global__ void __launch_bounds__(128, 2)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_w, const GemvArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  unsigned char* sa = smem;
  unsigned char* sb = smem + kStages * kTileA;
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(sb + kStages * kTileB);
  std::uint64_t* empty = full + kStages;
  std::uint64_t* done = empty + kStages;
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(done + 1);
  __shared__ RowDesc rds[kBM];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int live = a.meta ? __ldg(a.meta) : a.R;
  if (m0 >= live) return;  // uniform: the whole tile is past the live rows

  if (threadIdx.x == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_w);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc<kBN>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;
  const int kt_n = a.K / kBK;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kt = 0; kt < kt_n; ++kt) {
      const int s = kt % kStages;
      if (kt >= kStages) mbar_wait(&empty[s], ((kt / kStages) - 1) & 1);
      mbar_expect_tx(&full[s], kTileA + kTileB);
      tma_load_2d(sa + s * kTileA, &map_a, &full[s], kt * kBK, m0);
      tma_load_2d(sb + s * kTileB, &map_w, &full[s], kt * kBK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    for (int kt = 0; kt < kt_n; ++kt) {
      const int s = kt % kStages;
      mbar_wait(&full[s], (kt / kStages) & 1);
      tc_fence_after();
      const std::uint32_t a0 = smem_u32(sa + s * kTileA), b0 = smem_u32(sb + s * kTileB);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)  // K advance inside the 128-byte swizzle atom: +32 bytes
        umma_bf16(tmem, umma_desc(a0 + k * 32), umma_desc(b0 + k * 32), kIdesc, (kt | k) ? 1u : 0u);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();
  // ---- epilogue: thread = row m0 + 32*warp + lane; 16 columns per tcgen05.ld ----
  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < live;
  RowDesc rd{};
  if (row_ok && a.epi == kEpiQkv) {
    // while the main loop runs: this row's descriptor and its RoPE table row
    // into L1 (the epilogue reads one cos/sin pair per column pair)
    rd = a.rows[row];
    const char* rp = reinterpret_cast<const char*>(a.rope + static_cast<long long>(rd.pos) * (a.hd / 2));
    for (int off = 0; off < a.hd * 4; off += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(rp + off));
  }
  if (row_ok && a.epi == kEpiResidual) {  // the tile's residual row segment into L1 while the main loop runs
    const char* xp = reinterpret_cast<const char*>(a.out + static_cast<long long>(row) * a.N + n0);
    for (int off = 0; off < kBN * 4 && n0 + off / 4 < a.N; off += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(xp + off));
  }
  // normed linear map: the row's inverse RMS scales its fp32 products
  const float rs = (a.inv && row_ok) ? __ldcg(a.inv + row) : 1.f;
  mbar_wait(done, 0);
  tc_fence_after();
  // the QKV staging tile reuses the (now idle) pipeline smem
  block_epilogue(a, tmem + (static_cast<std::uint32_t>(warp * 32) << 16), row, row_ok, live, m0, n0, threadIdx.x, rd, rs,
                 reinterpret_cast<bf16*>(smem), rds, [] { __syncthreads(); });
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<kBN>(tmem);
}

// Persistent prompt-prefill GEMM: one CTA per SM, tiles t = blockIdx.x,
// blockIdx.x + gridDim.x, ... in M-fastest order over 128 x 256 tiles.
__global__ void __launch_bounds__(192, 1)
gemm_tc_persistent_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_w,
                          const GemvArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) & ~std::uintptr_t(1023));
  unsigned char* ring = smem;                                   // [kPStages][A 16 KB | W 32 KB]
  bf16* staging = reinterpret_cast<bf16*>(smem + kPStages * kPStage);
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kPStages * kPStage + kPStaging);
  std::uint64_t* empty = full + kPStages;
  std::uint64_t* acc_full = empty + kPStages;  // [2]: tile's accumulator complete
  std::uint64_t* acc_free = acc_full + 2;      // [2]: epilogue done reading it
  std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(acc_free + 2);
  __shared__ RowDesc rds[kBM];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int live = a.meta ? __ldg(a.meta) : a.R;
  const int mt = (live + kBM - 1) / kBM, nt = (a.N + kPN - 1) / kPN;
  const int tiles = mt * nt, kt_n = a.K / kBK;
  if (threadIdx.x == 0) {
    prefetch_tmap(&map_a);
    prefetch_tmap(&map_w);
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_free[b], 128);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: every tile's k-tiles through one ring ----
      int q = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t % mt) * kBM, n0 = (t / mt) * kPN;
        for (int kt = 0; kt < kt_n; ++kt, ++q) {
          const int s = q % kPStages;
          if (q >= kPStages) mbar_wait(&empty[s], ((q / kPStages) - 1) & 1);
          unsigned char* st = ring + s * kPStage;
          mbar_expect_tx(&full[s], kPStage);
          tma_load_2d(st, &map_a, &full[s], kt * kBK, m0);
          tma_load_2d(st + kTileA, &map_w, &full[s], kt * kBK, n0);
          tma_load_2d(st + kTileA + kPTileB / 2, &map_w, &full[s], kt * kBK, n0 + kPN / 2);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: tile i into accumulator i % 2 ----
      int q = 0, i = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int b = i & 1;
        if (i >= 2) mbar_wait(&acc_free[b], ((i >> 1) - 1) & 1);
        tc_fence_after();
        const std::uint32_t acc = tmem + b * kPN;
        for (int kt = 0; kt < kt_n; ++kt, ++q) {
          const int s = q % kPStages;
          mbar_wait(&full[s], (q / kPStages) & 1);
          tc_fence_after();
          const std::uint32_t a0 = smem_u32(ring + s * kPStage), b0 = a0 + kTileA;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            umma_bf16(acc, umma_desc(a0 + k * 32), umma_desc(b0 + k * 32), kPIdesc, (kt | k) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[b]);
      }
    }
  } else {
    // ---- epilogue warps 2-5: TMEM lane quarter = warp % 4 ----
    const int quarter = warp & 3, et = threadIdx.x - 64;
    int i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int b = i & 1;
      const int m0 = (t % mt) * kBM, n0 = (t / mt) * kPN;
      const int row = m0 + quarter * 32 + lane;
      const bool row_ok = row < live;
      const RowDesc rd = (row_ok && a.epi == kEpiQkv) ? a.rows[row] : RowDesc{};
      const float rs = (a.inv && row_ok) ? __ldcg(a.inv + row) : 1.f;
      mbar_wait(&acc_full[b], (i >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      const std::uint32_t tc = tmem + (static_cast<std::uint32_t>(quarter * 32) << 16) + b * kPN;
      for (int h = 0; h < kPN / kBN; ++h)
        block_epilogue(a, tc + h * kBN, row, row_ok, live, m0, n0 + h * kBN, et, rd, rs, staging, rds,
                       [] { asm volatile("bar.sync 1, 128;" ::: "memory"); });
      tc_fence_before();
      mbar_arrive(&acc_free[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Operand prep of a normed linear map, one CTA per row: h = bf16(x) and the
// row's inverse RMS (16-byte vector loads, block reduction in a fixed order).
__global__ void __launch_bounds__(128) rmsnorm_rows_kernel(const float* __restrict__ x, const int* __restrict__ sel,
                                                           const int* __restrict__ meta, int meta_idx, int K,
                                                           float* __restrict__ inv_out, float eps,
                                                           bf16* __restrict__ h) {
  __shared__ float red[4];
  __shared__ unsigned long long cst[kChainPhases];
  const int i = blockIdx.x;
  if (i >= meta[meta_idx]) return;  // tick metadata: not produced by the previous kernel
  const int r = sel ? sel[i] : i;
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) chain_mark(cst, 1);
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(r) * K);
  float ss = 0.f;
  for (int v = threadIdx.x; v < K / 4; v += 128) {
    const float4 t = xr[v];
    ss = fmaf(t.x, t.x, ss);
    ss = fmaf(t.y, t.y, ss);
    ss = fmaf(t.z, t.z, ss);
    ss = fmaf(t.w, t.w, ss);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float tot = red[0] + red[1] + red[2] + red[3];
  if (threadIdx.x == 0) inv_out[i] = 1.0f / sqrtf(tot / static_cast<float>(K) + eps);
  for (int v = threadIdx.x; v < K / 8; v += 128) {
    const float4 a = xr[2 * v], b = xr[2 * v + 1];
    __align__(16) bf16 o[8];
    o[0] = __float2bfloat16_rn(a.x);
    o[1] = __float2bfloat16_rn(a.y);
    o[2] = __float2bfloat16_rn(a.z);
    o[3] = __float2bfloat16_rn(a.w);
    o[4] = __float2bfloat16_rn(b.x);
    o[5] = __float2bfloat16_rn(b.y);
    o[6] = __float2bfloat16_rn(b.z);
    o[7] = __float2bfloat16_rn(b.w);
    reinterpret_cast<uint4*>(h + static_cast<long long>(i) * K)[v] = *reinterpret_cast<const uint4*>(o);
  }
  if (g_chain_stamp != nullptr) {
    __syncthreads();
    if (threadIdx.x == 0) {
      chain_mark(cst, 2);
      chain_flush(cst, 7u << 16);
    }
  }
}


using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

}  // namespace

bool make_tmap_bf16(TmaMap* out, const bf16* base, long long rows, long long cols, int box_rows) {
  static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "TmaMap must mirror CUtensorMap");
  EncodeFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(base),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool gemm_tc_supported(int N, int K) { return N % kBN == 0 && K % kBK == 0; }

void gemm_tc(const TmaMap& map_a, const TmaMap& map_w, const GemvArgs& a, cudaStream_t st) {
  if (a.R <= 0) return;
  static const bool persistent_on = [] {  // MOA_GEMM_PERSISTENT=0: the tile kernel for every M (A/B)
    const char* e = std::getenv("MOA_GEMM_PERSISTENT");
    return !(e && e[0] == '0');
  }();
  if (persistent_on && a.R > kPMinRows && a.N % kPN == 0) {
    static bool pattr = false;
    static int sms = 148;
    if (!pattr) {
      cudaFuncSetAttribute(gemm_tc_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem);
      uniform_carveout(reinterpret_cast<const void*>(gemm_tc_persistent_kernel));
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      pattr = true;
    }
    const int tiles = ((a.R + kBM - 1) / kBM) * (a.N / kPN);  // the row cap: live rows decide on the device
    gemm_tc_persistent_kernel<<<tiles < sms ? tiles : sms, 192, kPSmem, st>>>(
        *reinterpret_cast<const CUtensorMap*>(&map_a), *reinterpret_cast<const CUtensorMap*>(&map_w), a);
    return;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    uniform_carveout(reinterpret_cast<const void*>(gemm_tc_kernel));
    attr = true;
  }
  dim3 grid((a.N + kBN - 1) / kBN, (a.R + kBM - 1) / kBM);
  gemm_tc_kernel<<<grid, 128, kSmem, st>>>(*reinterpret_cast<const CUtensorMap*>(&map_a),
                                           *reinterpret_cast<const CUtensorMap*>(&map_w), a);
}

void rmsnorm_rows(const float* x, int R_cap, const int* meta, int K, float* inv, float eps, bf16* h,
                  cudaStream_t st, const int* sel, int meta_idx) {
  if (R_cap <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(R_cap);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  uniform_carveout(reinterpret_cast<const void*>(rmsnorm_rows_kernel));
  cudaLaunchKernelEx(&cfg, rmsnorm_rows_kernel, x, sel, meta, meta_idx, K, inv, eps, h);
}

MOA_CHAIN_STAMP_SETTER(gemm_tc_chain_stamp)

}  // namespace moa::k
