// Small device helpers: cache-policy loads, acquire/release flags, reductions.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace hxb {

// L2 policy for the once-streamed geometric factors: evict first, so the
// L-vectors (re-read across neighbouring element columns) stay in L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Non-volatile on purpose: the factors are immutable during a launch, so the
// compiler may hoist/batch these loads for latency hiding.
__device__ __forceinline__ double ld_stream(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

// One-instruction bulk prefetch of a contiguous block into L2 (TMA engine,
// sm_90+). Address and size must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ void prefetch_l2_bulk(const void* a, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(bytes) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Fixed-order block sum (warp shuffle tree, then warps in index order);
// the result is valid in thread 0 only. `red` holds NT/32 doubles.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];
  }
  __syncthreads();
  return s;
}

}  // namespace hxb
