// Debug only: per-CTA %globaltimer stamps of a tick's kernel chain
// (tools/chainstamp.py).  Off (one predicated load) while the buffer is null.
// A CTA keeps its stamps in shared memory and publishes them with a single
// atomic at its end, so stamping adds no global round trip inside the kernel.
// Buffer: [0] = record count, then (tag << 32 | phase << 24 | cta, ns) pairs.
#pragma once

namespace moa::k {
namespace {
// in constant memory: the "stamps off" test on every chain_mark is a
// constant-cache hit, not a global load on the kernel's critical path
__constant__ unsigned long long* g_chain_stamp = nullptr;
constexpr unsigned long long kChainStampCap = 1ull << 25;
constexpr int kChainPhases = 8;

__device__ __forceinline__ void chain_mark(unsigned long long* cs, int phase) {
  if (g_chain_stamp == nullptr) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  cs[phase] = t;
}

__device__ __forceinline__ void chain_reset(unsigned long long* cs) {
  if (g_chain_stamp == nullptr) return;
  for (int p = 0; p < kChainPhases; ++p) cs[p] = 0;
}

// call from one thread after every chain_mark of the CTA (fenced by a barrier)
__device__ __forceinline__ void chain_flush(const unsigned long long* cs, unsigned tag) {
  unsigned long long* b = g_chain_stamp;
  if (b == nullptr) return;
  int n = 0;
  for (int p = 0; p < kChainPhases; ++p) n += cs[p] != 0;
  const unsigned long long i0 = atomicAdd(b, static_cast<unsigned long long>(n));
  const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  unsigned long long i = i0;
  for (int p = 0; p < kChainPhases; ++p) {
    if (cs[p] == 0 || i >= kChainStampCap) continue;
    b[2 + 2 * i] = (static_cast<unsigned long long>(tag) << 32) | (static_cast<unsigned long long>(p) << 24) | cta;
    b[3 + 2 * i] = cs[p];
    ++i;
  }
}
}  // namespace
}  // namespace moa::k

// one setter per translation unit (the symbol above is TU-local)
#define MOA_CHAIN_STAMP_SETTER(fn) \
  void fn(unsigned long long* p) { cudaMemcpyToSymbol(g_chain_stamp, &p, sizeof(p)); }
