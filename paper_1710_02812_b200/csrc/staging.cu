// Staging copies that bypass the copy engines (see Staging in ctx.h).
#include "ctx.h"

namespace hsvdcu {

namespace {

__global__ void k_copy_mapped(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src,
                              size_t bytes) {
  const size_t n16 = bytes / 16;  // both ends 256-byte aligned (ring slots, arena blocks)
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x) d4[i] = s4[i];
  for (size_t i = n16 * 16 + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

}  // namespace

void copy_mapped_to_device(void* dst, const void* host_src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  k_copy_mapped<<<1, 256, 0, s>>>(static_cast<unsigned char*>(dst),
                                  static_cast<const unsigned char*>(host_src), bytes);
  HSVD_CUDA(cudaGetLastError());
}

}  // namespace hsvdcu
