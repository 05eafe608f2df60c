// Micro test (dev tool): 3D tiled tensor-map TMA of an 8x8x8 node block at
// arbitrary (odd) coordinates from a row-padded L-vector (row pitch even, so
// the strides are 16-byte multiples) into shared memory; checks the dense
// [z][y][x] layout and times back-to-back loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma3d tma3d.cu -lcuda && ./tma3d [smem offset bytes]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int NXP = 64, NX = 63, NY = 57, NZ = 40;

__device__ CUtensorMap g_tm;
__constant__ CUtensorMap c_tm;

__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int off_doubles, int mode) {
  const void* desc = mode == 0 ? static_cast<const void*>(&tm) : (mode == 1 ? static_cast<const void*>(&g_tm) : static_cast<const void*>(&c_tm));
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int x0 = (blockIdx.x * 7) % (NX - 7), y0 = (blockIdx.x * 5 + 3) % (NY - 7), z0 = (blockIdx.x * 3 + 1) % (NZ - 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(4096) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(s32(sm + off_doubles)),
        "l"(desc), "r"(x0), "r"(y0), "r"(z0), "r"(s32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(s32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[blockIdx.x * 512 + i] = sm[off_doubles + i];
}

int main(int argc, char** argv) {
  const int off = argc > 1 ? atoi(argv[1]) / 8 : 0;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const long long n = static_cast<long long>(NXP) * NY * NZ;
  std::vector<double> h(n);
  for (long long i = 0; i < n; ++i) h[i] = static_cast<double>(i);
  double *d, *o;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  const int blocks = 16;
  cudaMalloc(&o, blocks * 512 * 8);
  alignas(64) CUtensorMap tm;
  cuuint64_t dim[3] = {NX, NY, NZ};
  cuuint64_t gs[2] = {NXP * 8ull, static_cast<cuuint64_t>(NXP) * NY * 8};
  cuuint32_t box[3] = {8, 8, 8}, es[3] = {1, 1, 1};
  const int dt = argc > 3 ? atoi(argv[3]) : 0, l2 = argc > 4 ? atoi(argv[4]) : 1;
  const CUtensorMapDataType dts[3] = {CU_TENSOR_MAP_DATA_TYPE_FLOAT64, CU_TENSOR_MAP_DATA_TYPE_UINT64,
                                      CU_TENSOR_MAP_DATA_TYPE_INT64};
  const CUtensorMapL2promotion l2s[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
  printf("dtype %d l2 %d: ", dt, l2);
  CUresult cr = cuTensorMapEncodeTiled(&tm, dts[dt], 3, d, dim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_NONE, l2s[l2], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const char* es_ = nullptr;
  cuGetErrorString(cr, &es_);
  printf("encode: %d %s\n", static_cast<int>(cr), es_);
  if (cr != CUDA_SUCCESS) return 2;
  cudaMemcpyToSymbol(g_tm, &tm, sizeof tm);
  cudaMemcpyToSymbol(c_tm, &tm, sizeof tm);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<<<blocks, 128, 16384>>>(tm, o, off, mode);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> r(blocks * 512);
  cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int b = 0; b < blocks; ++b) {
    const int x0 = (b * 7) % (NX - 7), y0 = (b * 5 + 3) % (NY - 7), z0 = (b * 3 + 1) % (NZ - 7);
    for (int z = 0; z < 8; ++z)
      for (int y = 0; y < 8; ++y)
        for (int x = 0; x < 8; ++x)
          bad += r[b * 512 + (z * 8 + y) * 8 + x] != static_cast<double>((x0 + x) + NXP * ((y0 + y) + NY * (z0 + z)));
  }
  printf("mode %d smem offset %d B: err=%s mismatches=%d\n", mode, off * 8, cudaGetErrorString(e), bad);
  return e == cudaSuccess ? 0 : 1;
}
