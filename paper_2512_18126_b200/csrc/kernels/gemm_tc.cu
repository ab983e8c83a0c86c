// Prefill GEMM on the 5th-generation tensor cores (sm_100a):
//   Y[M][N] = A[M][K] . W[N][K]^T, bf16 operands, fp32 accumulation in TMEM.
//
// One CTA per 128 x 128 output tile, 4 warps:
//   warp 0 / lane 0  TMA producer: A and W k-tiles (64 x 128, SWIZZLE_128B)
//                    into a 4-stage shared-memory ring, mbarrier complete_tx;
//   warp 1 / lane 0  MMA issuer: tcgen05.mma.cta_group::1.kind::f16
//                    (M=128, N=128, K=16) x 4 per k-tile, tcgen05.commit
//                    frees the stage;
//   all 4 warps      epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes
//                    32w..32w+31 = rows), then the same epilogues as the GEMV
//                    path (RoPE + KV append, residual add, SwiGLU, fp32 store).
// With N along TMEM columns each thread holds consecutive columns of its row,
// so RoPE pairs and gate/up pairs (adjacent device columns) sit in one thread.
#include <cuda.h>

#include <cstdio>

#include "kernels.cuh"
#include "stamp.cuh"

namespace moa::k {

namespace {

// 128 x 128 tiles, 3 stages so two CTAs fit per SM and one CTA's epilogue
// overlaps the other's main loop (measured: C3 prefill GEMMs 252 -> 205 ms;
// 128 x 256 tiles with 2 stages lose on the small prefills of C1 / C2)
constexpr int kBM = 128, kBN = 128, kBK = 64, kStages = 3;
constexpr int kTileA = kBM * kBK * 2;  // 16 KB
constexpr int kTileB = kBN * kBK * 2;  // 16 KB
constexpr int kSmem = kStages * (kTileA + kTileB) + 1024 /*align*/ + 256 /*barriers*/;

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes));
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, std::uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, std::uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor: 8-row groups of
// 128-byte rows, SBO = 1024 B, LBO unused (1), version 1 (sm100), layout 2.
__device__ __forceinline__ std::uint64_t umma_desc(std::uint32_t saddr) {
  std::uint64_t d = 0;
  d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
  d |= static_cast<std::uint64_t>(1) << 16;
  d |= static_cast<std::uint64_t>(1024 >> 4) << 32;
  d |= static_cast<std::uint64_t>(1) << 46;
  d |= static_cast<std::uint64_t>(2) << 61;
  return d;
}

// kind::f16 instruction descriptor: F32 accumulate, BF16 A/B, K-major both.
constexpr std::uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<std::uint32_t>(kBN >> 3) << 17) |
                                 (static_cast<std::uint32_t>(kBM >> 4) << 24);

__device__ __forceinline__ void umma_f16(std::uint32_t tmem_d, std::uint64_t da, std::uint64_t db, std::uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(std::uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(std::uint32_t taddr, float (&v)[16]) {
  std::uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  const int live = a.meta ? __ldg(a.meta) : a.R;
  if (m0 >= live) return;  // uniform: the whole tile is past the live rows

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
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
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const std::uint32_t a0 = smem_u32(sa + s * kTileA), b0 = smem_u32(sb + s * kTileB);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)  // K advance inside the 128-byte swizzle atom: +32 bytes
        umma_f16(tmem, umma_desc(a0 + k * 32), umma_desc(b0 + k * 32), (kt | k) ? 1u : 0u);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();
  // ---- epilogue: thread = row m0 + 32*warp + lane; 16 columns per tcgen05.ld ----
  const int row = m0 + warp * 32 + lane;
  const bool row_ok = row < live;
  const std::uint32_t lane_base = static_cast<std::uint32_t>(warp * 32) << 16;
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
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  auto ld_scaled = [&](int c0, float (&v)[16]) {
    tmem_ld16(tmem + lane_base + static_cast<std::uint32_t>(c0), v);
    if (a.inv) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] *= rs;
    }
  };
  if (a.epi == kEpiQkv && kBN % a.hd == 0) {
    // RoPE + q / K / V rows staged as a bf16 tile in the (now idle) pipeline
    // smem in natural head order, then written out in 16-byte chunks: one
    // head row (hd x 2 bytes) per destination, instead of one 2-byte store per
    // element scattered over q and the KV pool
    bf16* st = reinterpret_cast<bf16*>(smem);  // [kBM][kBN], 16-byte chunks XOR-ed with row % 16
    // (a warp's threads are 32 rows writing the same column: without the
    // swizzle every store of a warp hits one bank)
    auto sti = [](int rr, int cc) { return rr * kBN + ((((cc >> 3) ^ (rr & 15))) << 3) + (cc & 7); };
    __shared__ RowDesc rds[kBM];
    rds[warp * 32 + lane] = rd;
    const int hd = a.hd, half = hd / 2, qk_cols = (a.nh + a.nkv) * hd;
    for (int c0 = 0; c0 < kBN; c0 += 16) {
      float v[16];
      ld_scaled(c0, v);
      if (!row_ok) continue;
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        const int n = n0 + c0 + i, cl = c0 + i;
        if (n < qk_cols) {
          const int e = (n % hd) / 2, hb = cl - (n % hd);  // tile-local head start
          const float2 cs = a.rope[static_cast<long long>(rd.pos) * half + e];
          const float x0 = v[i], x1 = v[i + 1];
          st[sti(warp * 32 + lane, hb + e)] = __float2bfloat16_rn(__fsub_rn(__fmul_rn(x0, cs.x), __fmul_rn(x1, cs.y)));
          st[sti(warp * 32 + lane, hb + e + half)] =
              __float2bfloat16_rn(__fadd_rn(__fmul_rn(x1, cs.x), __fmul_rn(x0, cs.y)));
        } else {
          st[sti(warp * 32 + lane, cl)] = __float2bfloat16_rn(v[i]);
          st[sti(warp * 32 + lane, cl + 1)] = __float2bfloat16_rn(v[i + 1]);
        }
      }
    }
    __syncthreads();
    const int cpr = kBN / 8;  // 16-byte chunks per tile row
    for (int c = threadIdx.x; c < kBM * cpr; c += 128) {
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
  } else
  for (int c0 = 0; c0 < kBN; c0 += 16) {
    float v[16];
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
      case kEpiQkv: {
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
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kBN));
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
