// Fused "U S V^T tile (+ X tile) -> sum of squares" kernel: the device form of
// the reference's chunked Frobenius evaluations (bench.cpp:30-42,
// svd_factor.cpp:66-80).  Summing squared pointwise differences avoids the
// cancellation a Gram-trace identity would suffer when the two operands
// nearly coincide (bench.cpp:27-29); nothing m x n is ever stored.
#include <algorithm>
#include <vector>

#include "metrics.h"

namespace hsvdcu {

namespace {

constexpr int TM = 64, TN = 64, TK = 16, NTH = 128;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename TX>
__device__ __forceinline__ double ldx(const TX* x, long long i) {
  return static_cast<double>(__ldg(x + i));
}

// One 64 x 64 tile of A B^T per CTA (4 warps x 32 x 32 DMMA blocks), then
// sum of (tile + X)^2 over the valid elements into part[tile].
template <typename TX>
__global__ void __launch_bounds__(NTH) k_prod_sumsq(const double* __restrict__ A, long long lda,
                                                    const double* __restrict__ B, long long ldb,
                                                    int m, int n, int k, const TX* __restrict__ X,
                                                    long long ldxx, double* __restrict__ part) {
  __shared__ double As[TK][TM + 4];
  __shared__ double Bs[TK][TN + 4];
  __shared__ double red[NTH / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < k; k0 += TK) {
    for (int e = tid; e < TM * TK; e += NTH) {  // m fastest: coalesced columns
      const int r = e % TM, kk = e / TM;
      const int gm = m0 + r, gk = k0 + kk;
      As[kk][r] = (gm < m && gk < k) ? A[gm + (long long)gk * lda] : 0.0;
      const int gn = n0 + r;
      Bs[kk][r] = (gn < n && gk < k) ? B[gn + (long long)gk * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk + tig][wm + i * 8 + grp];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk + tig][wn + j * 8 + grp];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int gm = m0 + wm + i * 8 + grp, gn = n0 + wn + j * 8 + 2 * tig + r;
        if (gm < m && gn < n) {
          double v = acc[i][j][r];
          if (X) v += ldx(X, (long long)gm * ldxx + gn);
          s += v * v;
        }
      }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NTH / 32; ++w) t += red[w];
    part[blockIdx.x + (long long)blockIdx.y * gridDim.x] = t;
  }
}

// Fixed-order reduction of the per-tile partials (one CTA).
__global__ void k_sum_parts(const double* __restrict__ part, long long count,
                            double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = threadIdx.x; i < count; i += blockDim.x) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// dst[:, c] = sign * w[c] * src[:, c] (w null: 1), column-major rows x cols
__global__ void k_scale_cols(double* __restrict__ dst, long long ldd, const double* __restrict__ src,
                             long long lds, int rows, int cols, const double* __restrict__ w,
                             double sign) {
  const long long total = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % rows), c = (int)(e / rows);
    dst[r + (long long)c * ldd] = sign * (w ? w[c] : 1.0) * src[r + (long long)c * lds];
  }
}

}  // namespace

void scale_cols_copy(Ctx& ctx, double* dst, long long ldd, const double* src, long long lds,
                     int rows, int cols, const double* w, double sign) {
  if (rows <= 0 || cols <= 0) return;
  const long long total = (long long)rows * cols;
  const int grid = (int)std::min<long long>((total + 255) / 256, 4096);
  ctx.launch_begin();
  k_scale_cols<<<grid, 256, 0, ctx.stream>>>(dst, ldd, src, lds, rows, cols, w, sign);
  ctx.check_launch("k_scale_cols");
}

double product_plus_sumsq(Ctx& ctx, const double* A, long long lda, const double* B,
                          long long ldb, int m, int n, int k, const void* X, DType dt,
                          long long ldxx) {
  if (m <= 0 || n <= 0) return 0.0;
  Arena::Mark mk = ctx.arena.mark();
  const dim3 grid(ceil_div(m, TM), ceil_div(n, TN));
  const long long tiles = (long long)grid.x * grid.y;
  double* part = ctx.arena.alloc_n<double>((size_t)tiles);
  double* d_out = ctx.arena.alloc_n<double>(1);
  ctx.launch_begin();
  if (!X || dt == DType::F64)
    k_prod_sumsq<double><<<grid, NTH, 0, ctx.stream>>>(A, lda, B, ldb, m, n, k,
                                                       static_cast<const double*>(X), ldxx, part);
  else
    k_prod_sumsq<float><<<grid, NTH, 0, ctx.stream>>>(A, lda, B, ldb, m, n, k,
                                                      static_cast<const float*>(X), ldxx, part);
  ctx.check_launch("k_prod_sumsq");
  ctx.launch_begin();
  k_sum_parts<<<1, 256, 0, ctx.stream>>>(part, tiles, d_out);
  ctx.check_launch("k_sum_parts");
  double* h = ctx.pinned_dbl(1);
  HSVD_CUDA(cudaMemcpyAsync(h, d_out, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
  const double r = h[0];
  ctx.arena.release(mk);
  return r;
}

}  // namespace hsvdcu
