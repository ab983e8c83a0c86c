// HBM-streaming decode GEMV for large weight matrices (sm_100a).
//
// y[r][n] = sum_k A[r][k] W[n][k] for R <= 8 rows (decode ticks).  One
// persistent CTA per SM; CTA b owns row groups g = b, b + grid, ... of 8
// weight rows.  A producer warp streams each group's rows in k-chunks of up to
// 2048 columns into a 4-stage shared-memory ring with cp.async.bulk
// (mbarrier complete_tx), keeping ~128 KB in flight per SM; 8 consumer warps
// (one per weight row of the group) dot the chunk against the activations,
// which are staged once per CTA in shared memory (normalised on the way in
// for the RMSNorm-prologue GEMMs).  Epilogues are the GEMV path's (RoPE + KV
// append, residual add, SwiGLU, fp32 store); pairs of adjacent weight rows
// (RoPE pairs, gate/up pairs) meet in shared memory.
#include <cstdio>

#include "kernels.cuh"

namespace moa::k {

namespace {

constexpr int kStages = 4;
constexpr int kConsumers = 8;    // consumer warps
constexpr int kGroup = 16;       // weight rows per group (an adjacent pair per consumer warp)
constexpr int kMaxKc = 1024;     // k-chunk columns (stage = 16 x 1024 bf16 = 32 KB)
constexpr int kAStageBytes = 64 * 1024;
constexpr int kThreads = 288;    // 8 consumer warps + 1 producer warp

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, std::uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)));
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float dot8_bf16(uint4 a, uint4 w, float acc) {
  const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 u = __bfloat1622float2(x[i]);
    const float2 v = __bfloat1622float2(y[i]);
    acc = fmaf(u.x, v.x, acc);
    acc = fmaf(u.y, v.y, acc);
  }
  return acc;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kThreads, 1) gemv_stream_kernel(const GemvArgs a, int kc) {
  extern __shared__ __align__(128) unsigned char smem[];
  bf16* As = reinterpret_cast<bf16*>(smem);                             // [R][K] (when staged)
  bf16* ring = reinterpret_cast<bf16*>(smem + kAStageBytes);           // [kStages][kGroup][kc]
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kAStageBytes + kStages * kGroup * kc * 2);
  std::uint64_t* empty = full + kStages;
  __shared__ float inv_s[8];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.meta ? __ldg(a.meta) : a.R;
  const int K = a.K, N = a.N;
  const int groups = (N + kGroup - 1) / kGroup;
  const int kchunks = K / kc;
  const bool staged = static_cast<long long>(R) * K * 2 <= kAStageBytes;
  if (R <= 0) return;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // stage the activations (bf16(x) for the RMSNorm-prologue GEMMs; inv_s scales their products)
  if (a.X && warp < R) {
    const float* xr = a.X + static_cast<long long>(warp) * K;
    float ss = 0.f;
    for (int k = lane * 4; k < K; k += 128) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(xr + k));
      ss = fmaf(v.x, v.x, ss);
      ss = fmaf(v.y, v.y, ss);
      ss = fmaf(v.z, v.z, ss);
      ss = fmaf(v.w, v.w, ss);
    }
    ss = warp_sum(ss);
    if (lane == 0) inv_s[warp] = 1.0f / sqrtf(ss / static_cast<float>(K) + a.eps);
  }
  __syncthreads();
  if (staged) {
    for (int i = threadIdx.x; i < R * K; i += kThreads) {
      const int r = i / K, k = i % K;
      As[i] = a.X ? __float2bfloat16_rn(a.X[static_cast<long long>(r) * K + k]) : a.A[static_cast<long long>(r) * K + k];
    }
  }
  __syncthreads();

  if (warp == kConsumers) {
    // ---- producer: stream weight row-slabs through the ring ----
    if (lane == 0) {
      int it = 0;
      for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        const int rows = min(kGroup, N - g * kGroup);
        const bf16* src0 = a.W + static_cast<long long>(g * kGroup) * K;
        for (int c = 0; c < kchunks; ++c, ++it) {
          const int s = it % kStages;
          if (it >= kStages) mbar_wait(&empty[s], ((it / kStages) - 1) & 1);
          mbar_expect_tx(&full[s], static_cast<std::uint32_t>(rows * kc * 2));
          bf16* dst = ring + static_cast<long long>(s) * kGroup * kc;
          if (kc == K) {  // the group's rows are one contiguous slab
            bulk_g2s(dst, src0, static_cast<std::uint32_t>(rows * kc * 2), &full[s]);
          } else {
            for (int r = 0; r < rows; ++r)
              bulk_g2s(dst + static_cast<long long>(r) * kc, src0 + static_cast<long long>(r) * K + c * kc,
                       static_cast<std::uint32_t>(kc * 2), &full[s]);
          }
        }
      }
    }
    return;
  }

  // ---- consumers: warp w owns the adjacent weight rows 2w, 2w+1 of a group ----
  int it = 0;
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    const int n0 = g * kGroup + 2 * warp;
    float acc0[8], acc1[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc0[r] = acc1[r] = 0.f;
    for (int c = 0; c < kchunks; ++c, ++it) {
      const int s = it % kStages;
      mbar_wait(&full[s], (it / kStages) & 1);
      if (n0 < N) {
        const bf16* w0 = ring + (static_cast<long long>(s) * kGroup + 2 * warp) * kc;
        const bf16* w1 = w0 + kc;
        const bool two = n0 + 1 < N;
        for (int k = lane * 8; k < kc; k += 256) {
          const uint4 u0 = *reinterpret_cast<const uint4*>(w0 + k);
          const uint4 u1 = two ? *reinterpret_cast<const uint4*>(w1 + k) : make_uint4(0, 0, 0, 0);
          const long long kk = static_cast<long long>(c) * kc + k;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            if (r < R) {
              const uint4 x = staged ? *reinterpret_cast<const uint4*>(As + r * K + kk)
                                     : __ldg(reinterpret_cast<const uint4*>(a.A + r * static_cast<long long>(K) + kk));
              acc0[r] = dot8_bf16(x, u0, acc0[r]);
              acc1[r] = dot8_bf16(x, u1, acc1[r]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (n0 >= N) continue;
    // reduce the R live rows; lane r then runs the epilogue for activation row r
    float v0 = 0.f, v1 = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < R) {
        const float s0 = warp_sum(acc0[r]), s1 = warp_sum(acc1[r]);
        if (lane == r) {
          v0 = s0;
          v1 = s1;
        }
      }
    }
    if (lane >= R) continue;
    const int r = lane;
    if (a.X) {  // RMSNorm on the fp32 product (the staged operand is bf16(x))
      v0 *= inv_s[r];
      v1 *= inv_s[r];
    }
    const bool two = n0 + 1 < N;
    switch (a.epi) {
      case kEpiF32:
        a.out[static_cast<long long>(r) * N + n0] = v0;
        if (two) a.out[static_cast<long long>(r) * N + n0 + 1] = v1;
        break;
      case kEpiResidual:
        a.out[static_cast<long long>(r) * N + n0] += v0;
        if (two) a.out[static_cast<long long>(r) * N + n0 + 1] += v1;
        break;
      case kEpiSwiGlu:  // rows 2j (gate) / 2j+1 (up)
        a.out_bf16[static_cast<long long>(r) * (N / 2) + n0 / 2] = __float2bfloat16_rn(v0 / (1.0f + __expf(-v0)) * v1);
        break;
      case kEpiQkv: {
        const RowDesc rd = a.rows[r];
        const int hd = a.hd, half = hd / 2, qk_cols = (a.nh + a.nkv) * hd;
        if (n0 < qk_cols) {  // RoPE pair (x0, x1) = rows (2i, 2i+1) of the head block
          const int head = n0 / hd, e = (n0 % hd) / 2;
          const float2 cs = a.rope[static_cast<long long>(rd.pos) * half + e];
          const float y0 = __fsub_rn(__fmul_rn(v0, cs.x), __fmul_rn(v1, cs.y));
          const float y1 = __fadd_rn(__fmul_rn(v1, cs.x), __fmul_rn(v0, cs.y));
          bf16* dst = head < a.nh ? a.out_bf16 + (static_cast<long long>(r) * a.nh + head) * hd
                                  : a.kpool + rd.kv * a.kv_stride + a.layer_off +
                                        (static_cast<long long>(head - a.nh) * a.max_ctx + rd.pos) * hd;
          dst[e] = __float2bfloat16_rn(y0);
          dst[e + half] = __float2bfloat16_rn(y1);
        } else {
          const int vc = n0 - qk_cols, kh = vc / hd, e = vc % hd;
          bf16* dst = a.vpool + rd.kv * a.kv_stride + a.layer_off + (static_cast<long long>(kh) * a.max_ctx + rd.pos) * hd + e;
          dst[0] = __float2bfloat16_rn(v0);
          dst[1] = __float2bfloat16_rn(v1);
        }
        break;
      }
    }
  }
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace

bool gemv_stream_supported(const GemvArgs& a) {
  // the RMSNorm prologue needs the staged activations (R x K bf16 <= 64 KB)
  const bool a_ok = !a.X || static_cast<long long>(a.R) * a.K * 2 <= kAStageBytes;
  return a.R <= 8 && (a.K % 256) == 0 && (a.N % 2) == 0 && a_ok &&
         static_cast<long long>(a.N) * a.K >= (4LL << 20);
}

void gemv_stream(const GemvArgs& a, cudaStream_t st) {
  int kc = a.K <= kMaxKc ? a.K : kMaxKc;  // largest multiple of 256 that divides K and fits a stage
  while (a.K % kc) kc -= 256;
  const int smem = kAStageBytes + kStages * kGroup * kc * 2 + 2 * kStages * 8;
  static int attr = 0;  // largest dynamic smem opted in so far
  if (smem > attr) {
    cudaFuncSetAttribute(gemv_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uniform_carveout(reinterpret_cast<const void*>(gemv_stream_kernel));
    attr = smem;
  }
  const int groups = (a.N + kGroup - 1) / kGroup;
  const int grid = groups < sm_count() ? groups : sm_count();
  gemv_stream_kernel<<<grid, kThreads, smem, st>>>(a, kc);
}

}  // namespace moa::k
