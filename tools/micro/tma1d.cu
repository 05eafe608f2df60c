// Micro test (dev tool): 1D tiled tensor-map TMA of 8-double rows at odd
// element offsets into shared-memory slots that are 16-byte but not 128-byte
// aligned, and into 128-byte aligned slots. Prints mismatches per mode.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma1d tma1d.cu -lcuda && ./tma1d
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int RANK>
__global__ void k(const __grid_constant__ CUtensorMap tm, double* out, int slot_stride, long long n) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ __align__(8) uint64_t bar;
  const int rows = 64;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(rows * 64) : "memory");
  __syncthreads();
  if (threadIdx.x < rows) {
    const int r = threadIdx.x;
    const int c = static_cast<int>((7 * (blockIdx.x * 64 + r) * 463LL + 3 * r + 1) % (n - 8));  // odd and even starts
    if (RANK == 1)
      asm volatile(
          "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
              s32(sm + r * slot_stride)),
          "l"(&tm), "r"(c), "r"(s32(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %4}], [%3];" ::"r"(
              s32(sm + r * slot_stride)),
          "l"(&tm), "r"(c), "r"(s32(&bar)), "r"(0)
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(s32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x)
    out[(blockIdx.x * rows) * 8 + i] = sm[(i / 8) * slot_stride + i % 8];
}

int main(int argc, char** argv) {
  const long long n = 463LL * 463 * 50;
  std::vector<double> h(n);
  for (long long i = 0; i < n; ++i) h[i] = static_cast<double>(i);
  double *d, *o;
  cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  const int blocks = 8;
  cudaMalloc(&o, blocks * 64 * 8 * 8);
  alignas(64) CUtensorMap tm;
  cuuint64_t dim[2] = {static_cast<cuuint64_t>(n), 1};
  cuuint64_t gs[1] = {static_cast<cuuint64_t>(n) * 8};
  cuuint32_t box[2] = {8, 1}, es[2] = {1, 1};
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  cuuint32_t rank = 1;
  for (int variant = 0; variant < 4 && cr != CUDA_SUCCESS; ++variant) {
    rank = variant < 2 ? 1 : 2;
    cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, d, dim, (variant & 1) ? gs : nullptr, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* es_ = nullptr;
    cuGetErrorString(cr, &es_);
    printf("encode variant %d (rank %u, strides %s): %d %s\n", variant, rank, (variant & 1) ? "set" : "null",
           static_cast<int>(cr), es_ ? es_ : "?");
  }
  if (cr != CUDA_SUCCESS) return 2;
  {
    const int stride = argc > 1 ? atoi(argv[1]) : 16;  // slot stride in doubles
    cudaMemset(o, 0, blocks * 64 * 8 * 8);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 68 * 8);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 68 * 8);
    if (rank == 1)
      k<1><<<blocks, 128, 64 * 68 * 8>>>(tm, o, stride, n);
    else
      k<2><<<blocks, 128, 64 * 68 * 8>>>(tm, o, stride, n);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> r(blocks * 64 * 8);
    cudaMemcpy(r.data(), o, r.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int b = 0; b < blocks; ++b)
      for (int row = 0; row < 64; ++row) {
        const long long c = (7 * (b * 64 + row) * 463LL + 3 * row + 1) % (n - 8);
        for (int i = 0; i < 8; ++i) bad += r[(b * 64 + row) * 8 + i] != static_cast<double>(c + i);
      }
    printf("slot stride %d doubles (%d B): err=%s mismatches=%d\n", stride, stride * 8, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
