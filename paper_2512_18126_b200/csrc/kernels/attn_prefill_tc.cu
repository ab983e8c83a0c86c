// Prompt-prefill attention on the 5th-generation tensor cores (K2 of SURVEY.md
// §2.2: the chunked-prefill attention of a prompt-prefill tick).
//
// CTA = one GQA group (kv head g) x P = 128 / hpg consecutive tick rows: its
// M = 128 MMA rows are the (row, q head) pairs of the group, so every K / V
// block the CTA loads serves all hpg heads.  FlashAttention dataflow on
// tcgen05 with both accumulators in TMEM:
//   warp 0   TMA producer: Q tile (3-D map over q [rows][nh][hd]), then the
//            64-key K and V blocks of each same-agent run through a 3-stage ring
//   warp 1   MMA issuer (one thread): S_j = Q.K_j^T into a double-buffered TMEM
//            S (M 128 x N 64); O += P_j.V_j into TMEM O (M 128 x N hd, V read
//            MN-major straight from the K/V pool layout)
//   warps 2-5  softmax: thread = TMEM lane = MMA row; S row by tcgen05.ld,
//            causal mask by the row's position, online softmax in log2 units,
//            P (bf16) into a 128B-swizzled smem tile, O row rescaled in TMEM
//            (tcgen05.ld / st) when its running max moves; final O / l -> bf16.
// Rows of the tick that are alone in their run (decode rows) are left to the
// per-row kernel; a row block spanning several agents' runs loops over the
// runs, each run's K / V streamed once (rows of other runs see p = 0).
//
// Key splits (incremental-prefill chunks: a tick of a few 32-row runs is only
// nkv x (rows / P) CTAs): grid.z = KS CTAs share a row block and form a
// thread-block cluster, each streaming a contiguous slice of every run's key
// blocks; each writes its rows' unnormalised O with the running reference m
// and the sum l (fp32) to a workspace (L2), and after one cluster barrier CTA
// s combines rows [s * 128 / KS, (s + 1) * 128 / KS) of the block from the KS
// partials in split order (O = sum 2^(m_s - M) O_s, l likewise; deterministic
// for a given tick shape).
//
// Algorithmic work per run of n rows ending at position p: causal
// Q.K^T and P.V over keys [0, p]: 4 * hd * (sum over rows of (pos + 1)) flops
// per q head; bytes: the run's keys once per kv head (K and V).
#include <cstdio>
#include <cstdlib>
#include <set>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "stamp.cuh"

namespace moa::k {
namespace {

using namespace tc;

constexpr unsigned kAll = 0xffffffffu;

template <int HD>
struct PfTc {
  static constexpr int KB = 64;                  // keys per block
  static constexpr int SUB = HD / 64;            // 64-column chunks of a row
  static constexpr int QCH = 128 * 128;          // one chunk of the Q tile: 128 rows x 128 B
  static constexpr int QB = SUB * QCH;
  static constexpr int KVCH = KB * 128;          // one chunk of a K or V block: 64 keys x 128 B
  static constexpr int STG = 3;
  static constexpr int STAGE = 2 * SUB * KVCH;   // K block + V block
  static constexpr int PB = 128 * KB * 2;        // P tile [128 rows][64 keys] bf16
  static constexpr int SMEM = 1024 + QB + STG * STAGE + 2 * PB;  // P double-buffered
  static constexpr int TMEM_COLS = 256;          // S0 | S1 | O
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// MN-major SWIZZLE_128B operand (V as the B operand of O += P.V: its rows are
// the K dimension, each 128-byte row holds 64 consecutive N elements): 8-row
// core groups SBO = 1024 B apart along K, 64-element atoms LBO apart along N.
__device__ __forceinline__ std::uint64_t umma_desc_mn(std::uint32_t saddr, std::uint32_t lbo) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<std::uint64_t>(1024 >> 4) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;
  d |= static_cast<std::uint64_t>(2) << 61;
  return d;
}

__device__ __forceinline__ void tmem_ld16_nw(std::uint32_t taddr, float* v) {
  std::uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(std::uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {  // 2^x on the SFU (ex2(-inf) = +0)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ std::uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const std::uint32_t*>(&v);
}

template <int HD>
__global__ void __launch_bounds__(192, 1)
attention_prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                            const __grid_constant__ CUtensorMap vmap, const RowDesc* __restrict__ rows,
                            const int* __restrict__ meta, int nh, int nkv, long long kv_stride, long long layer_off,
                            int max_ctx, bf16* __restrict__ o, float* __restrict__ ws) {
  using C = PfTc<HD>;
  constexpr int STG = C::STG, SUB = C::SUB;
  extern __shared__ unsigned char pt_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(pt_raw) + 1023) &
                                                       ~static_cast<std::uintptr_t>(1023));
  unsigned char* Qs = sm;                        // [SUB][128 rows][128 B]
  unsigned char* ring = Qs + C::QB;              // [STG][K: SUB x 64 keys x 128 B | V: same]
  unsigned char* Ps = ring + STG * C::STAGE;     // [2][128 rows][64 keys] bf16, 128B-swizzled
  // p_full alternates by item parity: the softmax warps may finish item i + 1
  // before the MMA thread observes item i's arrival (no rescale to wait for),
  // and a single barrier two phases ahead would alias the parity the MMA
  // thread waits on (a deadlock seen when other streams' kernels slow the
  // MMA thread down).  Every other barrier is bounded to one phase ahead.
  __shared__ __align__(8) std::uint64_t full[STG], empty[STG], q_full, s_full[2], s_free[2], p_full[2], o_done[2];
  __shared__ std::uint32_t tmem_slot;
  __shared__ RowDesc rd_s[128];
  __shared__ int seg_b[129], seg_e[128], seg_of[128];
  __shared__ int nseg_s, nitems_s, nblk_s[128], blk0_s[128];
  __shared__ unsigned long long cst[kChainPhases];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hpg = nh / nkv, P = 128 / hpg;
  const int b0 = blockIdx.x * P, g = blockIdx.y;
  const int KS = gridDim.z, split = blockIdx.z;
  const long long cl_blk = static_cast<long long>(blockIdx.x) * nkv + g;  // workspace slot of this row block
  const int live = __ldg(meta);
  if (b0 >= live) return;
  const int nb = min(P, live - b0);
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  // tick metadata (uploaded before the forward): runs of this row block
  if (threadIdx.x < nb) rd_s[threadIdx.x] = rows[b0 + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int i = 0; i < nb; ++i)
      if (i == 0 || rd_s[i].kv != rd_s[i - 1].kv || rd_s[i].pos != rd_s[i - 1].pos + 1) seg_b[n++] = i;
    seg_b[n] = nb;
    for (int i = 0; i < P; ++i) seg_of[i] = -1;
    int m = 0, items = 0;
    for (int k = 0; k < n; ++k) {
      const int a = seg_b[k], b = seg_b[k + 1];
      // a row alone in its run (its neighbours outside the block included) is a decode row
      const bool single = b - a == 1 && !(a == 0 && b0 > 0 && rows[b0 - 1].kv == rd_s[0].kv &&
                                            rows[b0 - 1].pos + 1 == rd_s[0].pos) &&
                          !(b == nb && b0 + nb < live && rows[b0 + nb].kv == rd_s[nb - 1].kv &&
                            rows[b0 + nb].pos == rd_s[nb - 1].pos + 1);
      if (single) continue;
      seg_b[m] = a;
      seg_e[m] = b;
      for (int i = a; i < b; ++i) seg_of[i] = m;
      const int tot = rd_s[b - 1].pos / C::KB + 1;  // keys [0, last position of the run]
      blk0_s[m] = split * tot / KS;  // this split's slice of them
      nblk_s[m] = (split + 1) * tot / KS - blk0_s[m];
      items += nblk_s[m];
      ++m;
    }
    nseg_s = m;
    nitems_s = items;
    for (int i = 0; i < STG; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&q_full, 1);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(&s_free[0], 128);
    mbar_init(&s_free[1], 128);
    mbar_init(&p_full[0], 128);
    mbar_init(&p_full[1], 128);
    mbar_init(&o_done[0], 1);
    mbar_init(&o_done[1], 1);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const std::uint32_t tmem = tmem_slot;
  const int nitems = nitems_s;
  pdl_wait();  // q, K and V of this tick are the QKV GEMM's outputs
  pdl_launch_dependents();
  if (threadIdx.x == 0) chain_mark(cst, 1);

  if (warp == 0) {
    if (lane == 0 && nitems > 0) {
      prefetch_tmap(&qmap);
      prefetch_tmap(&kmap);
      prefetch_tmap(&vmap);
      mbar_expect_tx(&q_full, C::QB);
      for (int c = 0; c < SUB; ++c) tma_load_3d(Qs + c * C::QCH, &qmap, &q_full, c * 64, g * hpg, b0);
      for (int sg = 0, i = 0; sg < nseg_s; ++sg)
      for (int j = 0; j < nblk_s[sg]; ++j, ++i) {
        const int st = i % STG;
        if (i >= STG) mbar_wait(&empty[st], ((i / STG) - 1) & 1);
        const RowDesc& r0 = rd_s[seg_b[sg]];
        const int row0 = static_cast<int>((r0.kv * kv_stride + layer_off) / HD + static_cast<long long>(g) * max_ctx) +
                         (blk0_s[sg] + j) * C::KB;
        mbar_expect_tx(&full[st], C::STAGE);
        unsigned char* kd = ring + st * C::STAGE;
#pragma unroll
        for (int c = 0; c < SUB; ++c) {
          tma_load_2d(kd + c * C::KVCH, &kmap, &full[st], c * 64, row0);
          tma_load_2d(kd + (SUB + c) * C::KVCH, &vmap, &full[st], c * 64, row0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nitems > 0) {
      constexpr std::uint32_t idS = idesc_bf16(128, C::KB);
      constexpr std::uint32_t idO = idesc_bf16(128, HD) | (1u << 16);  // B (V) MN-major
      const std::uint32_t q_u = smem_u32(Qs), p_u = smem_u32(Ps);
      mbar_wait(&q_full, 0);
      auto issue_s = [&](int i) {
        const int st = i % STG, sb = i & 1;
        mbar_wait(&full[st], (i / STG) & 1);
        if (i >= 2) mbar_wait(&s_free[sb], ((i >> 1) - 1) & 1);  // softmax of item i-2 read S[sb]
        tc_fence_after();
        const std::uint32_t k_u = smem_u32(ring + st * C::STAGE);
#pragma unroll
        for (int c = 0; c < SUB; ++c)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + sb * C::KB, umma_desc(q_u + c * C::QCH + k * 32), umma_desc(k_u + c * C::KVCH + k * 32),
                      idS, (c | k) ? 1u : 0u);
        umma_commit(&s_full[sb]);
      };
      issue_s(0);
      for (int i = 0; i < nitems; ++i) {
        if (i + 1 < nitems) issue_s(i + 1);
        mbar_wait(&p_full[i & 1], (i >> 1) & 1);  // P_i written, O rescaled
        tc_fence_after();
        const int st = i % STG;
        const std::uint32_t v_u = smem_u32(ring + st * C::STAGE + SUB * C::KVCH);
        const std::uint32_t pb_u = p_u + (i & 1) * C::PB;
#pragma unroll
        for (int k = 0; k < C::KB / 16; ++k)
          umma_bf16(tmem + 2 * C::KB, umma_desc(pb_u + k * 32), umma_desc_mn(v_u + k * 16 * 128, C::KVCH), idO,
                    (i | k) ? 1u : 0u);
        umma_commit(&o_done[i & 1]);
        umma_commit(&empty[st]);
      }
    }
  } else {
    // softmax warps: TMEM lane quarter = warp % 4, row = quarter * 32 + lane
    const int quarter = warp & 3, row = quarter * 32 + lane;
    const int pl = row / hpg, head = row % hpg;
    const int my_seg = pl < nb ? seg_of[pl] : -1;
    const int my_pos = pl < nb ? rd_s[pl].pos : -1;
    const std::uint32_t lane_off = static_cast<std::uint32_t>(quarter * 32) << 16;
    const std::uint32_t tS = tmem + lane_off, tO = tmem + lane_off + 2 * C::KB;
    const float sl2 = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;
    float m = -1e30f, l = 0.f;
    for (int sg = 0, i = 0; sg < nseg_s; ++sg)
    for (int j = 0; j < nblk_s[sg]; ++j, ++i) {
      const int sb = i & 1;
      mbar_wait(&s_full[sb], (i >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      float s[C::KB];
#pragma unroll
      for (int c = 0; c < C::KB / 16; ++c) tmem_ld16_nw(tS + sb * C::KB + c * 16, s + c * 16);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_free[sb]);
      const int kb = (blk0_s[sg] + j) * C::KB;
      const bool in = sg == my_seg;
      // causal mask only on blocks that reach past some row's position
      float mx = -INFINITY;
      if (__all_sync(kAll, in && kb + C::KB - 1 <= my_pos)) {
#pragma unroll
        for (int c = 0; c < C::KB; ++c) mx = fmaxf(mx, s[c]);
      } else {
#pragma unroll
        for (int c = 0; c < C::KB; ++c) {
          s[c] = (in && kb + c <= my_pos) ? s[c] : -INFINITY;
          mx = fmaxf(mx, s[c]);
        }
      }
      mx *= sl2;  // log2 units (sl2 > 0; -inf stays -inf)
      // Lazy rescaling: P is taken against the running reference m; only when
      // the block max exceeds it by more than 2^8 does the reference move (O
      // and l rescaled) -- P <= 256 is exact enough in bf16 (relative
      // rounding), and O / l cancels the reference.
      float alpha = 1.f;
      if (mx > m + 8.f) {
        alpha = ex2(m - mx);  // 0 while the row has seen no key (m = -1e30)
        m = mx;
      }
      const float nm = -m;
      float ps = 0.f;
#pragma unroll
      for (int c = 0; c < C::KB; ++c) {
        s[c] = ex2(fmaf(s[c], sl2, nm));  // masked keys: ex2(-inf) = 0
        ps += s[c];
      }
      l = l * alpha + ps;
      // P buffer i % 2 was last read by PV_{i-2}
      if (i >= 2) mbar_wait(&o_done[i & 1], ((i - 2) >> 1) & 1);
      unsigned char* prow = Ps + (i & 1) * C::PB + row * 128;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 v = make_uint4(pack2(s[8 * ch], s[8 * ch + 1]), pack2(s[8 * ch + 2], s[8 * ch + 3]),
                                   pack2(s[8 * ch + 4], s[8 * ch + 5]), pack2(s[8 * ch + 6], s[8 * ch + 7]));
        *reinterpret_cast<uint4*>(prow + ((ch ^ (row & 7)) << 4)) = v;
      }
      // rescale this row of O when its reference moved: after PV_{i-1}
      // (warp-collective TMEM access; rare after the first blocks)
      if (i > 0 && __any_sync(kAll, alpha != 1.f)) {
        mbar_wait(&o_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
        __syncwarp();
        tc_fence_after();
#pragma unroll
        for (int h2 = 0; h2 < HD / 64; ++h2) {
          float ov[64];
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_ld16_nw(tO + h2 * 64 + c * 16, ov + c * 16);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 64; ++k) ov[k] *= alpha;
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_st16(tO + h2 * 64 + c * 16, ov + c * 16);
        }
        tmem_wait_st();
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the tensor core
      tc_fence_before();
      mbar_arrive(&p_full[i & 1]);
    }
    if (KS > 1) {
      // key split: this row's partial (O relative to m, m, l) to the
      // workspace; combined below, after the cluster barrier
      float* wp = ws + ((cl_blk * KS + split) * 128 + row) * (HD + 4);
      if (nitems > 0) {
        mbar_wait(&o_done[(nitems - 1) & 1], ((nitems - 1) >> 1) & 1);
        __syncwarp();
        tc_fence_after();
      }
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        float ov[16];
        if (nitems > 0) {
          __syncwarp();
          tmem_ld16_nw(tO + c * 16, ov);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) ov[k] = 0.f;
        }
        float4* d4 = reinterpret_cast<float4*>(wp + c * 16);
#pragma unroll
        for (int k = 0; k < 4; ++k) __stcg(d4 + k, make_float4(ov[4 * k], ov[4 * k + 1], ov[4 * k + 2], ov[4 * k + 3]));
      }
      __stcg(reinterpret_cast<float4*>(wp + HD), make_float4(m, l, 0.f, 0.f));
    }
    if (KS == 1 && nitems > 0) {
      mbar_wait(&o_done[(nitems - 1) & 1], ((nitems - 1) >> 1) & 1);
      __syncwarp();
      tc_fence_after();
      // warp-collective TMEM loads (every lane), stores only for rows of a run
      const float inv = my_seg >= 0 ? 1.0f / l : 0.f;
      bf16* dst = o + (static_cast<long long>(b0 + pl) * nh + g * hpg + head) * HD;
#pragma unroll
      for (int c = 0; c < HD / 16; ++c) {
        float ov[16];
        __syncwarp();
        tmem_ld16_nw(tO + c * 16, ov);
        tmem_wait_ld();
        if (my_seg >= 0) {
          const uint4 a = make_uint4(pack2(ov[0] * inv, ov[1] * inv), pack2(ov[2] * inv, ov[3] * inv),
                                   pack2(ov[4] * inv, ov[5] * inv), pack2(ov[6] * inv, ov[7] * inv));
        const uint4 b = make_uint4(pack2(ov[8] * inv, ov[9] * inv), pack2(ov[10] * inv, ov[11] * inv),
                                   pack2(ov[12] * inv, ov[13] * inv), pack2(ov[14] * inv, ov[15] * inv));
          reinterpret_cast<uint4*>(dst + c * 16)[0] = a;
          reinterpret_cast<uint4*>(dst + c * 16)[1] = b;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (KS > 1) {
    // The KS CTAs of this row block form a cluster: once every partial is
    // written, CTA s combines rows [s * 128 / KS, (s + 1) * 128 / KS) of the
    // block, one float4 of a row's output per thread-item, summing the
    // partials in split order.
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int per = 128 / KS;
    const long long sstr = 128LL * (HD + 4);
    const float* base = ws + cl_blk * KS * sstr;
    for (int it = threadIdx.x; it < per * (HD / 4); it += blockDim.x) {
      const int r = split * per + it / (HD / 4), c4 = it % (HD / 4);
      const int pl = r / hpg, head = r % hpg;
      if (pl >= nb || seg_of[pl] < 0) continue;
      const float* rb = base + static_cast<long long>(r) * (HD + 4);
      float2 ml[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        ml[q] = q < KS ? __ldcg(reinterpret_cast<const float2*>(rb + q * sstr + HD)) : make_float2(-1e30f, 0.f);
      float4 t[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)
        t[q] = q < KS ? __ldcg(reinterpret_cast<const float4*>(rb + q * sstr) + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
      float M = -1e30f;
#pragma unroll
      for (int q = 0; q < 16; ++q) M = fmaxf(M, ml[q].x);
      float lt = 0.f;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q >= KS) break;
        const float sc = ex2(ml[q].x - M);
        lt += sc * ml[q].y;
        acc.x += sc * t[q].x;
        acc.y += sc * t[q].y;
        acc.z += sc * t[q].z;
        acc.w += sc * t[q].w;
      }
      const float inv = 1.0f / lt;
      bf16* dst = o + (static_cast<long long>(b0 + pl) * nh + g * hpg + head) * HD + 4 * c4;
      *reinterpret_cast<uint2*>(dst) = make_uint2(pack2(acc.x * inv, acc.y * inv), pack2(acc.z * inv, acc.w * inv));
    }
  }
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem);
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, (8u << 16) | 1u);
  }
}

}  // namespace

bool make_tmap_q3d(TmaMap* out, const bf16* q, long long rows, int nh, int hd, int hpg) {
  static_assert(sizeof(TmaMap) == sizeof(CUtensorMap), "TmaMap must mirror CUtensorMap");
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  if (!fn || 128 % hpg || hd % 64) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(hd), static_cast<cuuint64_t>(nh), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(hd) * 2, static_cast<cuuint64_t>(nh) * hd * 2};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(hpg), static_cast<cuuint32_t>(128 / hpg)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<bf16*>(q), dims,
            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Key splits per row block: only when the tick's grid (row blocks x kv heads)
// leaves most SMs idle, at least 2 key blocks per split, <= 8 splits (one
// portable cluster) and <=
// kPfTcMaxCtas CTAs in all (the workspace bound).
int attention_prefill_tc_splits(int R_cap, int nh, int nkv, int nblocks) {
  static const int cap = [] {  // MOA_PF_KSPLIT (A/B): max splits, 1 = off
    const char* e = std::getenv("MOA_PF_KSPLIT");
    return e ? std::max(1, std::min(8, std::atoi(e))) : 8;
  }();
  const int P = 128 / (nh / nkv);
  const int base = (R_cap + P - 1) / P * nkv;
  int KS = 1;
  while (KS * 2 <= cap && base * KS * 2 <= kPfTcMaxCtas && nblocks / (KS * 2) >= 2) KS *= 2;
  return KS;
}

long long attention_prefill_tc_ws_floats(int hd) { return static_cast<long long>(kPfTcMaxCtas) * 128 * (hd + 4); }

bool attention_prefill_tc_supported(int nh, int nkv, int hd) {
  return (hd == 64 || hd == 128) && nh % nkv == 0 && 128 % (nh / nkv) == 0 && nh / nkv <= 16;
}

void attention_prefill_tc(const TmaMap& qmap, const TmaMap& kmap, const TmaMap& vmap, const RowDesc* rows, int R_cap,
                          const int* meta, int nh, int nkv, int hd, long long kv_stride, long long layer_off,
                          int max_ctx, bf16* o, cudaStream_t st, int KS, float* ws) {
  if (R_cap <= 0) return;
  const int P = 128 / (nh / nkv);
  if (KS < 1 || KS > 8 || (KS > 1 && ((R_cap + P - 1) / P * nkv * KS > kPfTcMaxCtas || !ws))) {
    std::fprintf(stderr, "attention_prefill_tc: %d key splits exceed the workspace\n", KS);
    std::abort();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((R_cap + P - 1) / P, nkv, KS);
  cfg.blockDim = dim3(192);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (KS > 1) {  // the KS key splits of a row block: one cluster
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = KS;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  auto go = [&](auto kern, int smem) {
    static std::set<const void*> attr;
    if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      uniform_carveout(reinterpret_cast<const void*>(kern));
    }
    cfg.dynamicSmemBytes = smem;
    cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(&qmap),
                       *reinterpret_cast<const CUtensorMap*>(&kmap), *reinterpret_cast<const CUtensorMap*>(&vmap),
                       rows, meta, nh, nkv, kv_stride, layer_off, max_ctx, o, ws);
  };
  if (hd == 128)
    go(attention_prefill_tc_kernel<128>, PfTc<128>::SMEM);
  else
    go(attention_prefill_tc_kernel<64>, PfTc<64>::SMEM);
}

MOA_CHAIN_STAMP_SETTER(attn_prefill_tc_chain_stamp)

}  // namespace moa::k
