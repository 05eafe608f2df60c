// Micro test (dev tool): the triton probe's 2D fp64 TMA (64x64 tensor, 8x8 box) from CUDA C++.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

#ifdef WAITCTA
#define WSP "shared::cta"
#else
#define WSP "shared"
#endif
struct Big {
  double v[160];
};
template <int R>
__global__ void k(
#ifdef BIGPARAM
    const __grid_constant__ Big big,
#endif
    const __grid_constant__ CUtensorMap tm, double* out) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  double* sm = reinterpret_cast<double*>(smraw);
#ifdef STATICBAR
  __shared__ uint64_t sbar;
  uint64_t* bar = &sbar;
#else
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + 4096);
#endif
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)));
#ifdef FENCE
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef CTAEXP
#define EXPQ "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
#else
#define EXPQ "mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;"
#endif
    asm volatile(EXPQ ::"r"(s32(bar)), "r"(R == 2 ? 512 : 4096) : "memory");
    if (R == 2)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              s32(sm)),
          "l"(&tm), "r"(16), "r"(8), "r"(s32(bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %5}], [%4];" ::"r"(
              s32(sm)),
#ifdef DYNCOORD
          "l"(&tm), "r"(16 + (int)(blockIdx.x % 3)), "r"(8 - (int)(blockIdx.x % 2)), "r"(s32(bar)), "r"(3 - (int)(blockIdx.x & 1))
#else
          "l"(&tm), "r"(16), "r"(8), "r"(s32(bar)), "r"(3)
#endif
          : "memory");
  }
#ifndef NOSYNC
  __syncthreads();
#endif
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity." WSP ".b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(s32(bar))
      : "memory");
  if (threadIdx.x < 64) out[threadIdx.x] = sm[threadIdx.x];
}

int main(int argc, char** argv) {
  const int sw = argc > 1 ? atoi(argv[1]) : 0, rank = argc > 2 ? atoi(argv[2]) : 2;
  std::vector<double> h(64 * 57 * 40);
  for (int i = 0; i < 64 * 57 * 40; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, 64 * 57 * 40 * 8);
  cudaMalloc(&o, 64 * 8);
  cudaMemcpy(d, h.data(), 64 * 57 * 40 * 8, cudaMemcpyHostToDevice);
  alignas(64) CUtensorMap tm;
  const int dx = argc > 3 ? atoi(argv[3]) : 64;
#ifdef T3DIMS
  cuuint64_t dim[3] = {63, 57, 40}, gs[2] = {512, 64 * 57 * 8};
#else
  cuuint64_t dim[3] = {static_cast<cuuint64_t>(dx), rank == 2 ? 64ull : 16ull, 4}, gs[2] = {512, 16 * 512};
#endif
  cuuint32_t box[3] = {8, 8, 8}, es[3] = {1, 1, 1};
  CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, d, dim, gs, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       sw ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d; ", static_cast<int>(cr));
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
#ifdef BIGPARAM
  Big big{};
  if (rank == 2) k<2><<<1, 128, 8192>>>(big, tm, o); else k<3><<<1, 128, 8192>>>(big, tm, o);
#else
#ifdef MANY
  if (rank == 2) k<2><<<16, 128, 8192>>>(tm, o); else k<3><<<16, 128, 8192>>>(tm, o);
#else
  if (rank == 2) k<2><<<1, 128, 8192>>>(tm, o); else k<3><<<1, 128, 8192>>>(tm, o);
#endif
#endif
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> r(64);
  cudaMemcpy(r.data(), o, 64 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 8; ++x) bad += r[y * 8 + x] != h[(rank == 3 ? 3 * 16 * 64 : 0) + (8 + y) * 64 + 16 + x];
  printf("rank %d swizzle %d: %s, mismatches %d\n", rank, sw, cudaGetErrorString(e), bad);
  return 0;
}
