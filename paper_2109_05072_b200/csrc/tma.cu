// TMA tensor maps for the u staging of the DMMA operator kernels.
//
// The reference's L-vector is unpadded (mesh.hpp:40-46): node (X, Y, Z) at
// X + Nx (Y + Ny Z), so with Nx odd (every box mesh with an even element count
// along x) its row stride is not the 16-byte multiple a tensor map needs. The
// single-GPU fast CG therefore keeps its search direction p row-pitched
// (Workspace::pt, pitch = Nx rounded up to even); the operator kernel then
// stages each element's (p+1)^3 node block -- the gather of
// restriction.hpp:55-65 / operator.hpp:223-225 -- with ONE
// cp.async.bulk.tensor.3d per element instead of (p+1)^2 row copies.
// Applies on caller vectors (unpadded) keep the cp.async path.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "internal.h"

namespace hxb {

bool use_mma(const Setup& s);  // apply.cu

bool tma_u_supported(const Setup& s) { return use_mma(s) && s.p == 7; }

// HEXBP_NO_TMA_U=1 (dev A/B and the bitwise test): same row-pitched vectors,
// u staged by cp.async instead of the tensor copy
bool tma_u_staging_enabled() {
  static const bool off = std::getenv("HEXBP_NO_TMA_U") != nullptr;
  return !off;
}

int tma_u_pitch(const Setup& s) { return (s.dims[0] * s.p + 1 + 1) & ~1; }

cudaError_t encode_u_tensor_map(const Setup& s, const double* u, int pitch, CUtensorMap* map) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (enc == nullptr) return cudaErrorNotSupported;
  const int n = s.p + 1;
  const cuuint64_t Nx = static_cast<cuuint64_t>(s.dims[0]) * s.p + 1, Ny = static_cast<cuuint64_t>(s.dims[1]) * s.p + 1,
                   Nz = static_cast<cuuint64_t>(s.dims[2]) * s.p + 1;
  if ((pitch & 1) || static_cast<cuuint64_t>(pitch) < Nx || (reinterpret_cast<uintptr_t>(u) & 15)) return cudaErrorInvalidValue;
  const cuuint64_t dim[3] = {static_cast<cuuint64_t>(pitch), Ny, Nz};  // the pad column is part of the rows
  const cuuint64_t stride[2] = {static_cast<cuuint64_t>(pitch) * 8, static_cast<cuuint64_t>(pitch) * Ny * 8};
  // A box row must start 16-byte aligned (an odd fp64 start coordinate faults):
  // the kernels load n + 2 doubles from the even x at or below the element's
  // first node (x = 7 ex is odd for odd ex).
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(n + 2), static_cast<cuuint32_t>(n), static_cast<cuuint32_t>(n)};
  const cuuint32_t es[3] = {1, 1, 1};
  static const int l2 = [] {  // L2 fetch granularity (dev A/B switch HEXBP_TMA_L2 = 0..3: none, 64, 128, 256 B)
    const char* v = std::getenv("HEXBP_TMA_L2");
    return v ? std::atoi(v) & 3 : 2;
  }();
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(u), dim, stride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         static_cast<CUtensorMapL2promotion>(l2), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

}  // namespace hxb
