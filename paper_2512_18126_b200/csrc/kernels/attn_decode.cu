// Decode attention for GQA agents (one query row per agent; K3 of SURVEY.md
// §2.2): the row's KV prefix is cut into fixed splits of KEYS keys, one CTA
// per (row, kv head, split).  A CTA stages its whole split of K and V with
// TMA (64-key boxes, 128B-swizzled, 64-column subtiles) behind one mbarrier:
// boxes below the first key written in this tick are issued before the
// programmatic-dependent-launch wait (the previous kernel of the chain writes
// the keys of this tick's rows: `pos`, and the earlier rows of an agent's
// incremental-prefill run), so the KV stream overlaps the QKV GEMV's tail.  The
// group's q heads are the M rows of mma.sync m16n8k16 tiles; each of the 4
// warps takes KEYS/4 keys: S = Q.K^T, masked online softmax on the fragments,
// O += P.V with V^T fragments from ldmatrix.trans; the warps combine in smem in
// a fixed order and a row spanning several splits is combined by the
// last-arriving CTA in split order (deterministic for given shapes).
//
// Algorithmic bytes per (row, kv head): (pos + 1) * hd * 2 (K) * 2 (V).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <set>

#include "kernels.cuh"
#include "mma_common.cuh"
#include "tc_common.cuh"
#include "stamp.cuh"

namespace moa::k {
namespace {

using namespace tc;

constexpr unsigned kAll = 0xffffffffu;

template <int HD>
struct DecTma {
  static constexpr int KEYS = HD == 128 ? 128 : 256;  // keys per CTA (one split)
  static constexpr int KW = KEYS / 4;                 // keys per warp
  static constexpr int SUB = HD / 64;                 // 64-column (128 B) subtiles per key row
  static constexpr int KVB = KEYS * HD * 2;           // bytes of K (or V) per CTA
  static constexpr int QB = 16 * HD * 2;              // Q tile
  static constexpr int SMEM = 1024 + 2 * KVB + QB + 64;
};

template <int HD>
__global__ void __launch_bounds__(128)
attention_decode_tma_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                            const bf16* __restrict__ q, const RowDesc* __restrict__ rows, const int* __restrict__ meta,
                            int nh, int nkv, long long kv_stride, long long layer_off, int max_ctx,
                            bf16* __restrict__ o, float* __restrict__ ws, int* __restrict__ cnt, int nsplit_max,
                            int skip_runs) {
  using C = DecTma<HD>;
  constexpr int KW = C::KW, NJ = KW / 8, KSTEPS = HD / 16, NT = HD / 8, RB = HD * 2;
  extern __shared__ unsigned char dt_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(dt_raw) + 1023) &
                                                       ~static_cast<std::uintptr_t>(1023));
  unsigned char* Ks = sm;                // [SUB][KEYS][128 B], TMA 128B swizzle
  unsigned char* Vs = sm + C::KVB;       // same
  unsigned char* Qs = sm + 2 * C::KVB;   // [16][HD] bf16, 16-byte chunks XOR-swizzled by row
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(Qs + C::QB);
  float* wo = reinterpret_cast<float*>(Ks);  // after the key loop: [4 warps][16][HD] fp32
  __shared__ float wm[4][16], wl[4][16], cm_s[16], cl_s[16];
  __shared__ bool last;
  __shared__ unsigned long long cst[kChainPhases];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int r = blockIdx.x, g = blockIdx.y, s = blockIdx.z;
  const int live = __ldg(meta);  // tick metadata: uploaded before the forward
  if (r >= live) return;
  const RowDesc rd = rows[r];
  if (skip_runs) {
    if ((r > 0 && rows[r - 1].kv == rd.kv && rows[r - 1].pos + 1 == rd.pos) ||
        (r + 1 < live && rows[r + 1].kv == rd.kv && rows[r + 1].pos == rd.pos + 1))
      return;
  }
  const int n = rd.pos + 1;
  const int nsplit = (n + C::KEYS - 1) / C::KEYS;
  if (s >= nsplit) return;
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  const int hpg = nh / nkv;
  const int kb = s * C::KEYS, ke = min(n, kb + C::KEYS);
  const int nbox = (ke - kb + 63) / 64;
  // First key written in this tick: the row's own key, or the first key of the
  // run of consecutive rows of the same agent it ends (incremental-prefill
  // rows of one agent share a tick and see each other's keys).  Warp 0 walks
  // back 32 rows per step (tick metadata: readable before the PDL wait).
  int first_new = rd.pos;
  if (warp == 0) {
    int base = r - 1, p = rd.pos - 1;
    for (;;) {
      const int rr = base - lane;
      const bool c = rr >= 0 && rows[rr].kv == rd.kv && rows[rr].pos == p - lane;
      const unsigned b = __ballot_sync(kAll, c);
      if (b == kAll) {
        base -= 32;
        p -= 32;
        continue;
      }
      first_new = p - (__ffs(~b) - 1) + 1;
      break;
    }
  }
  // boxes from this one on hold keys the previous kernel writes: issued after the wait
  const int newbox = first_new < ke ? max(0, first_new - kb) / 64 : nbox;
  const int row0 = static_cast<int>((rd.kv * kv_stride + layer_off) / HD + static_cast<long long>(g) * max_ctx + kb);
  auto load_box = [&](int b) {
#pragma unroll
    for (int sub = 0; sub < C::SUB; ++sub) {
      tma_load_2d(Ks + sub * (C::KEYS * 128) + b * 64 * 128, &kmap, full, sub * 64, row0 + b * 64);
      tma_load_2d(Vs + sub * (C::KEYS * 128) + b * 64 * 128, &vmap, full, sub * 64, row0 + b * 64);
    }
  };
  if (threadIdx.x == 0) {
    prefetch_tmap(&kmap);
    prefetch_tmap(&vmap);
    mbar_init(full, 1);
    mbar_fence_init();
    mbar_expect_tx(full, static_cast<std::uint32_t>(nbox * C::SUB * 2 * 64 * 128));
    for (int b = 0; b < newbox; ++b) load_box(b);  // keys of earlier ticks: not written by the previous kernel
  }
  pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    chain_mark(cst, 1);
    for (int b = newbox; b < nbox; ++b) load_box(b);
  }
  for (int c = threadIdx.x; c < 16 * (HD / 8); c += 128) {
    const int hr = c / (HD / 8), ch = c % (HD / 8);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (hr < hpg) v = __ldcg(reinterpret_cast<const uint4*>(q + (static_cast<long long>(r) * nh + g * hpg + hr) * HD) + ch);
    *reinterpret_cast<uint4*>(Qs + hr * RB + ((ch ^ (hr & 7)) << 4)) = v;
  }
  __syncthreads();
  const std::uint32_t qs_u = smem_u32(Qs), ks_u = smem_u32(Ks), vs_u = smem_u32(Vs);
  std::uint32_t qa[KSTEPS][4];
#pragma unroll
  for (int kk = 0; kk < KSTEPS; ++kk) {
    const int hr = lane & 15, ch = kk * 2 + (lane >> 4);
    ldsm_x4(qs_u + hr * RB + ((ch ^ (hr & 7)) << 4), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
  }
  // element (key row kr, 16-byte chunk ch of the HD row) in a TMA-swizzled K / V stage
  auto kv_addr = [](std::uint32_t base, int kr, int ch) {
    return base + (ch >> 3) * (C::KEYS * 128) + kr * 128 + (((ch & 7) ^ (kr & 7)) << 4);
  };
  const float sl2 = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;
  float m_a = -1e30f, m_b = -1e30f, l_a = 0.f, l_b = 0.f;
  float oacc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) oacc[nt][0] = oacc[nt][1] = oacc[nt][2] = oacc[nt][3] = 0.f;
  const int wk0 = warp * KW;  // this warp's first key (relative to kb)
  mbar_wait(full, 0);
  if (threadIdx.x == 0) chain_mark(cst, 3);
  if (kb + wk0 < ke) {
    float sacc[NJ][4];
#pragma unroll
    for (int j = 0; j < NJ; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
#pragma unroll
      for (int jp = 0; jp < NJ / 2; ++jp) {
        const int kr = wk0 + jp * 16 + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        std::uint32_t b00, b01, b10, b11;
        ldsm_x4(kv_addr(ks_u, kr, ch), b00, b01, b10, b11);
        mma_bf16(sacc[2 * jp], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b00, b01);
        mma_bf16(sacc[2 * jp + 1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b10, b11);
      }
    }
    float mx_a = -1e30f, mx_b = -1e30f;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int key = kb + wk0 + 8 * j + 2 * t4;
      sacc[j][0] = key < ke ? sacc[j][0] * sl2 : -1e30f;
      sacc[j][1] = key + 1 < ke ? sacc[j][1] * sl2 : -1e30f;
      sacc[j][2] = key < ke ? sacc[j][2] * sl2 : -1e30f;
      sacc[j][3] = key + 1 < ke ? sacc[j][3] * sl2 : -1e30f;
      mx_a = fmaxf(mx_a, fmaxf(sacc[j][0], sacc[j][1]));
      mx_b = fmaxf(mx_b, fmaxf(sacc[j][2], sacc[j][3]));
    }
    mx_a = fmaxf(mx_a, __shfl_xor_sync(kAll, mx_a, 1));
    mx_a = fmaxf(mx_a, __shfl_xor_sync(kAll, mx_a, 2));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(kAll, mx_b, 1));
    mx_b = fmaxf(mx_b, __shfl_xor_sync(kAll, mx_b, 2));
    m_a = mx_a;
    m_b = mx_b;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      sacc[j][0] = sacc[j][0] <= -1e29f ? 0.f : exp2f(sacc[j][0] - m_a);
      sacc[j][1] = sacc[j][1] <= -1e29f ? 0.f : exp2f(sacc[j][1] - m_a);
      sacc[j][2] = sacc[j][2] <= -1e29f ? 0.f : exp2f(sacc[j][2] - m_b);
      sacc[j][3] = sacc[j][3] <= -1e29f ? 0.f : exp2f(sacc[j][3] - m_b);
      l_a += sacc[j][0] + sacc[j][1];
      l_b += sacc[j][2] + sacc[j][3];
    }
    // O = P V over this warp's keys: P (16 x KW) from the S fragments
#pragma unroll
    for (int kk = 0; kk < KW / 16; ++kk) {
      const std::uint32_t pa0 = pack_bf16(sacc[2 * kk][0], sacc[2 * kk][1]);
      const std::uint32_t pa1 = pack_bf16(sacc[2 * kk][2], sacc[2 * kk][3]);
      const std::uint32_t pa2 = pack_bf16(sacc[2 * kk + 1][0], sacc[2 * kk + 1][1]);
      const std::uint32_t pa3 = pack_bf16(sacc[2 * kk + 1][2], sacc[2 * kk + 1][3]);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int vr = wk0 + kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = np * 2 + (lane >> 4);
        std::uint32_t v00, v01, v10, v11;
        ldsm_x4_t(kv_addr(vs_u, vr, ch), v00, v01, v10, v11);
        mma_bf16(oacc[2 * np], pa0, pa1, pa2, pa3, v00, v01);
        mma_bf16(oacc[2 * np + 1], pa0, pa1, pa2, pa3, v10, v11);
      }
    }
  }
  l_a += __shfl_xor_sync(kAll, l_a, 1);
  l_a += __shfl_xor_sync(kAll, l_a, 2);
  l_b += __shfl_xor_sync(kAll, l_b, 1);
  l_b += __shfl_xor_sync(kAll, l_b, 2);
  __syncthreads();  // every warp is done reading K / V (wo reuses the K stage)
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
  if (threadIdx.x < hpg) {  // warp combine, fixed order
    const int h = threadIdx.x;
    float M = -1e30f;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w][h]);
    float Lsum = 0.f;
    for (int w = 0; w < 4; ++w) Lsum += wl[w][h] == 0.f ? 0.f : exp2f(wm[w][h] - M) * wl[w][h];
    cm_s[h] = M;
    cl_s[h] = Lsum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < hpg * HD; i += 128) {
    const int h = i / HD, e = i % HD;
    const float M = cm_s[h];
    float val = 0.f;
    for (int w = 0; w < 4; ++w)
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
  if (nsplit == 1) {
    if (g_chain_stamp != nullptr && threadIdx.x == 0) {
      chain_mark(cst, 2);
      chain_flush(cst, (6u << 16) | 1u);
    }
    return;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(cnt + r * nkv + g) : "memory");
    last = prev == static_cast<unsigned>(nsplit - 1);
  }
  __syncthreads();
  if (!last) {
    if (g_chain_stamp != nullptr && threadIdx.x == 0) {
      chain_mark(cst, 2);
      chain_flush(cst, (6u << 16) | 1u);
    }
    return;
  }
  // combine the splits in split order
  float* sw_s = reinterpret_cast<float*>(Vs);  // [16][64] split weights
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
  if (threadIdx.x == 0) {
    cnt[r * nkv + g] = 0;
    chain_mark(cst, 2);
    chain_flush(cst, (6u << 16) | 1u);
  }
}


// ---------------------------------------------------------------------------
// Cluster-split decode attention.  The row's keys are cut into NS splits of
// whole 64-key boxes; the NS CTAs of one (row, kv head) form a thread-block
// cluster (grid x = split).  A producer warp streams the split's boxes (K and
// V, 128B-swizzled TMA) through an STG-stage mbarrier ring; the four consumer
// warps take 16 keys of every box each (q heads of the GQA group = the M rows
// of mma.sync m16n8k16 tiles) with an online softmax across boxes, so loads
// overlap compute and a CTA holds only STG boxes.  Partials are combined
// without global memory: each CTA folds its warps (fixed order) into
// (max, sum, o) and pushes each slice of o, with every head's (max, sum), into
// the owning rank's landing buffer with st.async (DSMEM stores completing on
// the owner's mbarrier); CTA s waits only for its own slice and combines the
// ranks in rank order (deterministic for given shapes).  NS = 8 for every row
// (a row's splits depend only on its context length: batch invariant); two
// ring stages per CTA suffice with 8 kv heads x 8 splits per row in flight
// and leave room on the SM for the next GEMV's CTAs (PDL prologue).
template <int HD, int STG_ = (HD == 128 ? 2 : 3)>
struct DecCl {
  static constexpr int STG = STG_;                 // ring stages (64-key boxes of K and V)
  static constexpr int SUB = HD / 64;              // 128-byte column subtiles per key row
  static constexpr int BOX = 64 * HD * 2;          // bytes of one K (or V) box
  static constexpr int STAGE = 2 * BOX;
  static constexpr int QB = 16 * HD * 2;
  static constexpr int WO = 4 * 16 * HD * 4;       // warp partials (reuse the ring)
  static_assert(WO <= STG * STAGE, "warp partials fit in the ring");
  static constexpr int SMEM = 1024 + STG * STAGE + QB + 2 * STG * 8;
};

template <int HD, int STG_>
__global__ void __launch_bounds__(160)
attention_decode_cluster_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                                const bf16* __restrict__ q, const RowDesc* __restrict__ rows,
                                const int* __restrict__ meta, int nh, int nkv, long long kv_stride,
                                long long layer_off, int max_ctx, bf16* __restrict__ o, int skip_runs) {
  using C = DecCl<HD, STG_>;
  constexpr int KSTEPS = HD / 16, NT = HD / 8, RB = HD * 2, STG = C::STG;
  extern __shared__ unsigned char dc_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(dc_raw) + 1023) &
                                                       ~static_cast<std::uintptr_t>(1023));
  unsigned char* ring = sm;                    // [STG][K box | V box], each [SUB][64][128 B] swizzled
  unsigned char* Qs = sm + STG * C::STAGE;     // [16][HD] bf16, 16-byte chunks XOR-swizzled by row
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(Qs + C::QB);
  std::uint64_t* empty = full + STG;
  float* wo = reinterpret_cast<float*>(ring);  // after the box loop: [4 warps][16][HD]
  __shared__ float wm[4][16], wl[4][16];
  // partials pushed here by every rank of the cluster (st.async): this CTA's
  // slice of the outputs [NS][chunk] and every rank's (max, sum) per q head
  __shared__ __align__(16) float land_o[8 * 256];
  __shared__ __align__(16) float land_ml[16 * 16 * 2];
  __shared__ __align__(8) std::uint64_t land_bar;
  __shared__ int first_new_s;
  __shared__ unsigned long long cst[kChainPhases];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g8 = lane >> 2, t4 = lane & 3;
  const int s = blockIdx.x, NS = gridDim.x, g = blockIdx.y, r = blockIdx.z;
  // cluster-uniform early exits (every CTA of a cluster has the same row)
  const int live = __ldg(meta);
  if (r >= live) return;
  const RowDesc rd = rows[r];
  if (skip_runs) {
    if ((r > 0 && rows[r - 1].kv == rd.kv && rows[r - 1].pos + 1 == rd.pos) ||
        (r + 1 < live && rows[r + 1].kv == rd.kv && rows[r + 1].pos == rd.pos + 1))
      return;
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    chain_reset(cst);
    chain_mark(cst, 0);
  }
  const int hpg = nh / nkv;
  const int n = rd.pos + 1, nbox = (n + 63) / 64, bps = (nbox + NS - 1) / NS;
  const int b0 = min(nbox, s * bps), nb = min(nbox, b0 + bps) - b0;
  if (warp == 4) {
    // First key written in this tick: the row's own, or the first of the run
    // of consecutive rows of its agent it ends (incremental-prefill rows of one
    // agent share a tick); boxes from there on are issued after the PDL wait.
    int base = r - 1, p = rd.pos - 1, fn = rd.pos;
    for (;;) {
      const int rr = base - lane;
      const bool c = rr >= 0 && rows[rr].kv == rd.kv && rows[rr].pos == p - lane;
      const unsigned b = __ballot_sync(kAll, c);
      if (b == kAll) {
        base -= 32;
        p -= 32;
        continue;
      }
      fn = p - (__ffs(~b) - 1) + 1;
      break;
    }
    if (lane == 0) {
      first_new_s = fn;
      for (int i = 0; i < STG; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 4);
      }
      mbar_init(&land_bar, 1);
      const int chunk = hpg * HD / NS;
      mbar_expect_tx(&land_bar, static_cast<std::uint32_t>(NS * (chunk * 4 + hpg * 8)));
      mbar_fence_init();
    }
  }
  __syncthreads();
  // this CTA's landing barrier is armed (peers wait for it before pushing)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (warp == 4) {
    if (lane == 0) {
      prefetch_tmap(&kmap);
      prefetch_tmap(&vmap);
      const int newbox = first_new_s / 64;  // absolute index of the first box holding a new key
      const int row0 = static_cast<int>((rd.kv * kv_stride + layer_off) / HD + static_cast<long long>(g) * max_ctx);
      bool waited = false;
      for (int i = 0; i < nb; ++i) {
        const int st = i % STG, b = b0 + i;
        if (i >= STG) mbar_wait(&empty[st], ((i / STG) - 1) & 1);
        if (!waited && b >= newbox) {
          pdl_wait();
          waited = true;
        }
        mbar_expect_tx(&full[st], C::STAGE);
        unsigned char* kd = ring + st * C::STAGE;
#pragma unroll
        for (int sub = 0; sub < C::SUB; ++sub) {
          tma_load_2d(kd + sub * 8192, &kmap, &full[st], sub * 64, row0 + b * 64);
          tma_load_2d(kd + C::BOX + sub * 8192, &vmap, &full[st], sub * 64, row0 + b * 64);
        }
      }
    }
  } else {
    pdl_wait();  // q is written by the previous kernel
    if (threadIdx.x == 0) chain_mark(cst, 1);
    for (int c = threadIdx.x; c < 16 * (HD / 8); c += 128) {
      const int hr = c / (HD / 8), ch = c % (HD / 8);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (hr < hpg) v = __ldcg(reinterpret_cast<const uint4*>(q + (static_cast<long long>(r) * nh + g * hpg + hr) * HD) + ch);
      *reinterpret_cast<uint4*>(Qs + hr * RB + ((ch ^ (hr & 7)) << 4)) = v;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // consumer warps only
  }
  float m_a = -1e30f, m_b = -1e30f, l_a = 0.f, l_b = 0.f;
  float oacc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) oacc[nt][0] = oacc[nt][1] = oacc[nt][2] = oacc[nt][3] = 0.f;
  if (warp < 4) {
    const std::uint32_t qs_u = smem_u32(Qs);
    std::uint32_t qa[KSTEPS][4];
#pragma unroll
    for (int kk = 0; kk < KSTEPS; ++kk) {
      const int hr = lane & 15, ch = kk * 2 + (lane >> 4);
      ldsm_x4(qs_u + hr * RB + ((ch ^ (hr & 7)) << 4), qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3]);
    }
    // element (key row kr, 16-byte chunk ch of the HD row) of a swizzled box
    auto kv_addr = [](std::uint32_t base, int kr, int ch) {
      return base + (ch >> 3) * 8192 + kr * 128 + (((ch & 7) ^ (kr & 7)) << 4);
    };
    const float sl2 = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;
    const int wk = warp * 16;  // this warp's 16 keys of every box
    for (int i = 0; i < nb; ++i) {
      const int st = i % STG;
      const int kb = (b0 + i) * 64 + wk;  // absolute key of this warp's first key
      const std::uint32_t ks_u = smem_u32(ring + st * C::STAGE), vs_u = ks_u + C::BOX;
      mbar_wait(&full[st], (i / STG) & 1);
      if (i == 0 && threadIdx.x == 0) chain_mark(cst, 3);
      float sacc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KSTEPS; ++kk) {
        const int kr = wk + (lane & 7) + ((lane >> 4) << 3);
        const int ch = kk * 2 + ((lane >> 3) & 1);
        std::uint32_t b00, b01, b10, b11;
        ldsm_x4(kv_addr(ks_u, kr, ch), b00, b01, b10, b11);
        mma_bf16(sacc[0], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b00, b01);
        mma_bf16(sacc[1], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b10, b11);
      }
      float mx_a = -1e30f, mx_b = -1e30f;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int key = kb + 8 * j + 2 * t4;
        sacc[j][0] = key < n ? sacc[j][0] * sl2 : -1e30f;
        sacc[j][1] = key + 1 < n ? sacc[j][1] * sl2 : -1e30f;
        sacc[j][2] = key < n ? sacc[j][2] * sl2 : -1e30f;
        sacc[j][3] = key + 1 < n ? sacc[j][3] * sl2 : -1e30f;
        mx_a = fmaxf(mx_a, fmaxf(sacc[j][0], sacc[j][1]));
        mx_b = fmaxf(mx_b, fmaxf(sacc[j][2], sacc[j][3]));
      }
      mx_a = fmaxf(mx_a, __shfl_xor_sync(kAll, mx_a, 1));
      mx_a = fmaxf(mx_a, __shfl_xor_sync(kAll, mx_a, 2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(kAll, mx_b, 1));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(kAll, mx_b, 2));
      const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
      const float al_a = exp2f(m_a - mn_a), al_b = exp2f(m_b - mn_b);
      m_a = mn_a;
      m_b = mn_b;
      l_a *= al_a;
      l_b *= al_b;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        oacc[nt][0] *= al_a;
        oacc[nt][1] *= al_a;
        oacc[nt][2] *= al_b;
        oacc[nt][3] *= al_b;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        sacc[j][0] = sacc[j][0] <= -1e29f ? 0.f : exp2f(sacc[j][0] - m_a);
        sacc[j][1] = sacc[j][1] <= -1e29f ? 0.f : exp2f(sacc[j][1] - m_a);
        sacc[j][2] = sacc[j][2] <= -1e29f ? 0.f : exp2f(sacc[j][2] - m_b);
        sacc[j][3] = sacc[j][3] <= -1e29f ? 0.f : exp2f(sacc[j][3] - m_b);
        l_a += sacc[j][0] + sacc[j][1];
        l_b += sacc[j][2] + sacc[j][3];
      }
      const std::uint32_t pa0 = pack_bf16(sacc[0][0], sacc[0][1]);
      const std::uint32_t pa1 = pack_bf16(sacc[0][2], sacc[0][3]);
      const std::uint32_t pa2 = pack_bf16(sacc[1][0], sacc[1][1]);
      const std::uint32_t pa3 = pack_bf16(sacc[1][2], sacc[1][3]);
#pragma unroll
      for (int np = 0; np < NT / 2; ++np) {
        const int vr = wk + (lane & 7) + (((lane >> 3) & 1) << 3);
        const int ch = np * 2 + (lane >> 4);
        std::uint32_t v00, v01, v10, v11;
        ldsm_x4_t(kv_addr(vs_u, vr, ch), v00, v01, v10, v11);
        mma_bf16(oacc[2 * np], pa0, pa1, pa2, pa3, v00, v01);
        mma_bf16(oacc[2 * np + 1], pa0, pa1, pa2, pa3, v10, v11);
      }
      // the stage's generic-proxy reads (ldmatrix) are ordered before the
      // producer's next TMA (async-proxy) write into it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    l_a += __shfl_xor_sync(kAll, l_a, 1);
    l_a += __shfl_xor_sync(kAll, l_a, 2);
    l_b += __shfl_xor_sync(kAll, l_b, 1);
    l_b += __shfl_xor_sync(kAll, l_b, 2);
  }
  __syncthreads();  // every box consumed: the ring is free for the partials
  if (threadIdx.x == 0) chain_mark(cst, 4);
  if (warp < 4) {
    if (t4 == 0) {
      wm[warp][g8] = m_a;
      wl[warp][g8] = l_a;
      wm[warp][g8 + 8] = m_b;
      wl[warp][g8 + 8] = l_b;
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int d = nt * 8 + 2 * t4;
      *reinterpret_cast<float2*>(wo + (warp * 16 + g8) * HD + d) = make_float2(oacc[nt][0], oacc[nt][1]);
      *reinterpret_cast<float2*>(wo + (warp * 16 + g8 + 8) * HD + d) = make_float2(oacc[nt][2], oacc[nt][3]);
    }
  }
  __syncthreads();
  // This CTA's partial over its boxes (warps folded in a fixed order), pushed
  // straight into the owners' landing buffers: rank q owns output elements
  // [q * chunk, (q + 1) * chunk) of the group's hpg x HD outputs.
  const int chunk = hpg * HD / NS;
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every landing barrier is armed
  if (threadIdx.x == 0) chain_mark(cst, 5);
  for (int t = threadIdx.x; t < hpg * HD / 4; t += blockDim.x) {
    const int e0 = 4 * t, h = e0 / HD, e = e0 % HD;
    float M = -1e30f;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w][h]);
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < 4; ++w)
      if (wl[w][h] != 0.f) {
        const float c = exp2f(wm[w][h] - M);
        const float4 x = *reinterpret_cast<const float4*>(wo + (w * 16 + h) * HD + e);
        val.x += c * x.x;
        val.y += c * x.y;
        val.z += c * x.z;
        val.w += c * x.w;
      }
    const int q = e0 / chunk, off = e0 % chunk;
    std::uint32_t dst, bar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(land_o + s * chunk + off)), "r"(q));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(&land_bar)), "r"(q));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(dst),
                 "f"(val.x), "f"(val.y), "f"(val.z), "f"(val.w), "r"(bar)
                 : "memory");
  }
  for (int t = threadIdx.x; t < NS * hpg; t += blockDim.x) {
    const int q = t / hpg, h = t % hpg;
    float M = -1e30f;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w][h]);
    float L = 0.f;
    for (int w = 0; w < 4; ++w) L += wl[w][h] == 0.f ? 0.f : exp2f(wm[w][h] - M) * wl[w][h];
    std::uint32_t dst, bar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(dst) : "r"(smem_u32(land_ml + (s * hpg + h) * 2)), "r"(q));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(smem_u32(&land_bar)), "r"(q));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(dst),
                 "f"(M), "f"(L), "r"(bar)
                 : "memory");
  }
  // rank s combines its slice over all ranks, in rank order
  mbar_wait(&land_bar, 0);
  for (int i = threadIdx.x; i < chunk; i += blockDim.x) {
    const int e = s * chunk + i, h = e / HD;
    float M = -1e30f;
    for (int t = 0; t < NS; ++t) M = fmaxf(M, land_ml[(t * hpg + h) * 2]);
    float L = 0.f, val = 0.f;
    for (int t = 0; t < NS; ++t) {
      const float lt = land_ml[(t * hpg + h) * 2 + 1];
      const float w = lt == 0.f ? 0.f : exp2f(land_ml[(t * hpg + h) * 2] - M);
      L += w * lt;
      val += w * land_o[t * chunk + i];
    }
    o[(static_cast<long long>(r) * nh + g * hpg) * HD + e] = __float2bfloat16_rn(val / L);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    chain_mark(cst, 2);
    chain_flush(cst, (6u << 16) | 1u);
  }
}

}  // namespace

MOA_CHAIN_STAMP_SETTER(attn_decode_chain_stamp)

int attention_decode_tma_keys(int hd) { return hd == 128 ? DecTma<128>::KEYS : DecTma<64>::KEYS; }

bool attention_decode_tma_supported(int nh, int nkv, int hd, int max_ctx) {
  return (hd == 64 || hd == 128) && nh % nkv == 0 && nh / nkv <= 16 &&
         (max_ctx + attention_decode_tma_keys(hd) - 1) / attention_decode_tma_keys(hd) <= 64;
}

void attention_decode_tma(const TmaMap& kmap, const TmaMap& vmap, const bf16* q, const RowDesc* rows, int R_cap,
                          int nsplit_cap, const int* meta, int nh, int nkv, int hd, long long kv_stride,
                          long long layer_off, int max_ctx, bf16* o, float* ws, int* cnt, cudaStream_t st,
                          bool skip_runs) {
  if (R_cap <= 0) return;
  const int nsplit_max = (max_ctx + kKvSplit - 1) / kKvSplit;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(R_cap, nkv, nsplit_cap);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  auto go = [&](auto kern, int smem) {
    static std::set<const void*> attr;
    if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      uniform_carveout(reinterpret_cast<const void*>(kern));
    }
    cfg.dynamicSmemBytes = smem;
    cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(&kmap),
                       *reinterpret_cast<const CUtensorMap*>(&vmap), q, rows, meta, nh, nkv, kv_stride, layer_off,
                       max_ctx, o, ws, cnt, nsplit_max, skip_runs ? 1 : 0);
  };
  if (hd == 128)
    go(attention_decode_tma_kernel<128>, DecTma<128>::SMEM);
  else
    go(attention_decode_tma_kernel<64>, DecTma<64>::SMEM);
}


int attention_decode_cluster_splits(int rcap, int nkv, int nbox_cap) {
  // Fixed: a row's split structure (and so its accumulation order) depends
  // only on its own context length, never on the tick's row count -- schedule
  // modes that batch rows differently decode identical tokens.
  (void)rcap, (void)nkv, (void)nbox_cap;
  static const int ns = [] {  // MOA_ATTN_SPLITS (A/B): 8 (portable cluster) or 16 (non-portable)
    const char* e = std::getenv("MOA_ATTN_SPLITS");
    return e && std::atoi(e) == 16 ? 16 : 8;
  }();
  return ns;
}

bool attention_decode_cluster_supported(int nh, int nkv, int hd) {
  return (hd == 64 || hd == 128) && nh % nkv == 0 && nh / nkv <= 16;
}

void attention_decode_cluster(const TmaMap& kmap, const TmaMap& vmap, const bf16* q, const RowDesc* rows, int R_cap,
                              int ns, const int* meta, int nh, int nkv, int hd, long long kv_stride,
                              long long layer_off, int max_ctx, bf16* o, cudaStream_t st, bool skip_runs) {
  if (R_cap <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ns, nkv, R_cap);
  cfg.blockDim = dim3(160);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ns;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  auto go = [&](auto kern, int smem) {
    static std::set<const void*> attr;
    if (attr.insert(reinterpret_cast<const void*>(kern)).second) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      uniform_carveout(reinterpret_cast<const void*>(kern));
    }
    cfg.dynamicSmemBytes = smem;
    cudaLaunchKernelEx(&cfg, kern, *reinterpret_cast<const CUtensorMap*>(&kmap),
                       *reinterpret_cast<const CUtensorMap*>(&vmap), q, rows, meta, nh, nkv, kv_stride, layer_off,
                       max_ctx, o, skip_runs ? 1 : 0);
  };
  static const int stg = [] {  // MOA_ATTN_STAGES=3: a 3-stage ring for hd 128 (A/B)
    const char* e = std::getenv("MOA_ATTN_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  if (hd == 128 && stg == 3)
    go(attention_decode_cluster_kernel<128, 3>, DecCl<128, 3>::SMEM);
  else if (hd == 128)
    go(attention_decode_cluster_kernel<128, 2>, DecCl<128, 2>::SMEM);
  else
    go(attention_decode_cluster_kernel<64, 3>, DecCl<64, 3>::SMEM);
}

}  // namespace moa::k
