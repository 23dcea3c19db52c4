// Shared device/host helpers for the B200 HSVD library (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace hsvdcu {

// Status codes mirrored in include/hsvd_cu.h.
enum Status : int {
  kOk = 0,
  kInvalid = 1,      // std::invalid_argument in the reference
  kDecomposition = 2,  // hsvd::DecompositionError in the reference
  kCuda = 3,
  kNccl = 4,
  kNoMemory = 5,
  kIo = 6,      // hsvd::IoError in the reference (matrix_io.hpp)
  kFormat = 7,  // hsvd::FormatError in the reference (matrix_io.hpp)
};

struct Error : std::runtime_error {
  Error(int code, const std::string& what, long long rows = 0, long long cols = 0)
      : std::runtime_error(what), code(code), rows(rows), cols(cols) {}
  int code;
  long long rows, cols;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

#define HSVD_CUDA(x) ::hsvdcu::cuda_check((x), #x)

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

#ifdef __CUDACC__
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block-wide sum (fixed reduction tree). `red` needs
// blockDim.x/32 doubles of shared memory. All threads receive the result.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  return t;
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double t = lane < nw ? red[lane] : -1.0e308;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  double r = red[0];
  return r;
}

template <typename T>
__device__ __forceinline__ double to_f64(T v) { return static_cast<double>(v); }
#endif

}  // namespace hsvdcu
