// Per-factor finalisation and small helper kernels.
//
// finalize() turns projected directions P = A z_i into an SvdFactor slice:
// sigma_i = ||A z_i||_2 (column norms carry relative accuracy eps*kappa, not
// the eps*kappa^2 of sqrt(lambda_i)), sorted non-increasing, truncated with
// the reference rule keep = min(retained_count(sigma, gamma), max_rank)
// (svd_factor.cpp:23-46, merge.cpp:106-109), degenerate = (sigma_1 == 0)
// (svd_factor.cpp:25,44, merge.cpp:115-116).  Directions with sigma below
// 1e-6*sigma_1 cannot be normalised stably; they are completed to an
// orthonormal set by Gram-Schmidt, as the reference's SVD kernels return an
// orthonormal U for rank-deficient inputs.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "factor_ops.h"

namespace hsvdcu {

namespace {

constexpr int FIN_THREADS = 256;

__global__ void __launch_bounds__(FIN_THREADS) k_finalize(const FinJob* __restrict__ jobs) {
  const FinJob J = jobs[blockIdx.x];
  const int s = J.s, p = J.p;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  extern __shared__ double sm[];
  double* sig_old = sm;
  double* sig_new = sig_old + p;
  double* dots = sig_new + p;
  double* red = dots + p;
  int* perm = reinterpret_cast<int*>(red + 32);
  int* bad = perm + p;
  __shared__ int s_keep, s_write;
  __shared__ double s_smax;

  // 1. column norms
  __shared__ int s_nan;
  if (tid == 0) s_nan = 0;
  for (int i = tid; i < p; i += nt) perm[i] = i;
  __syncthreads();
  for (int c = warp; c < p; c += nwarps) {
    const double* col = J.P + (long long)c * J.ldp;
    double acc = 0.0;
    if (J.norms2) {
      acc = J.norms2[c];
    } else {
      for (int r = lane; r < s; r += 32) acc += col[r] * col[r];
      acc = warp_sum(acc);
    }
    if (lane == 0) {
      double v = sqrt(acc);
      if (!isfinite(v)) {
        v = -1.0;
        s_nan = 1;
      }
      sig_old[c] = v;
    }
  }
  __syncthreads();
  // 2. stable descending rank sort
  for (int c = tid; c < p; c += nt) {
    const double v = sig_old[c];
    int pos = 0;
    for (int c2 = 0; c2 < p; ++c2) {
      const double w = sig_old[c2];
      pos += (w > v) || (w == v && c2 < c);
    }
    perm[pos] = c;
    sig_new[pos] = v;
  }
  __syncthreads();
  // 3. truncation count
  if (tid == 0) {
    const double smax = sig_new[0];
    int keep;
    int deg = 0;
    if (s_nan) {
      keep = 1;
      deg = 2;  // non-finite input: reported as a decomposition failure
    } else if (smax == 0.0) {
      keep = 1;
      deg = 1;
    } else {
      const double cutoff = J.gamma * smax;
      keep = 0;
      while (keep < p && sig_new[keep] >= cutoff) ++keep;
      if (keep < 1) keep = 1;
    }
    if (J.cap > 0 && keep > J.cap) keep = J.cap;
    s_keep = keep;
    s_write = J.write_all ? p : keep;
    s_smax = smax;
    *J.rank = keep;
    *J.degenerate = deg;
  }
  __syncthreads();
  const int wr = s_write;
  const double smax = s_smax;
  for (int i = tid; i < p; i += nt) {
    J.sigma[i] = sig_new[i];
    if (J.perm) J.perm[i] = perm[i];
    bad[i] = !(sig_new[i] > 1e-6 * smax) || smax == 0.0;
  }
  __syncthreads();
  // 4. normalised columns
  for (int i = 0; i < wr; ++i) {
    const double* src = J.P + (long long)perm[i] * J.ldp;
    double* dst = J.U + (long long)i * J.ldu;
    double inv = bad[i] ? 1.0 : 1.0 / sig_new[i];
    if (J.norms2) inv = sig_new[i] > 0.0 ? 1.0 / sig_new[i] : 0.0;
    for (int r = tid; r < s; r += nt) dst[r] = src[r] * inv;
  }
  __syncthreads();
  if (J.norms2) return;  // sharded: completion would need a global Gram-Schmidt
  // 5. complete unstable / null directions (rare: rank-deficient inputs)
  for (int i = 0; i < wr; ++i) {
    if (!bad[i]) continue;
    double* ui = J.U + (long long)i * J.ldu;
    int attempt = 0;
    double pre = 0.0;
    {
      double part = 0.0;
      for (int r = tid; r < s; r += nt) part += ui[r] * ui[r];
      pre = block_sum(part, red);
    }
    while (true) {
      if (pre == 0.0 || !isfinite(pre)) {
        const int e = (i + attempt) % s;
        for (int r = tid; r < s; r += nt) ui[r] = (r == e) ? 1.0 : 0.0;
        pre = 1.0;
        ++attempt;
        __syncthreads();
      }
      for (int rep = 0; rep < 2; ++rep) {
        for (int j = warp; j < wr; j += nwarps) {
          double acc = 0.0;
          if (j != i && (!bad[j] || j < i)) {
            const double* uj = J.U + (long long)j * J.ldu;
            for (int r = lane; r < s; r += 32) acc += uj[r] * ui[r];
            acc = warp_sum(acc);
          }
          if (lane == 0) dots[j] = acc;
        }
        __syncthreads();
        for (int r = tid; r < s; r += nt) {
          double a = ui[r];
          for (int j = 0; j < wr; ++j)
            if (dots[j] != 0.0) a -= dots[j] * J.U[r + (long long)j * J.ldu];
          ui[r] = a;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int r = tid; r < s; r += nt) part += ui[r] * ui[r];
      const double post = block_sum(part, red);
      if (post > 1e-2 * pre && post > 0.0) {
        const double sc = 1.0 / sqrt(post);
        for (int r = tid; r < s; r += nt) ui[r] *= sc;
        __syncthreads();
        break;
      }
      if (attempt > s) break;  // cannot happen for wr <= s
      pre = 0.0;               // take the next unit vector
      __syncthreads();
    }
  }
}

__global__ void k_scale_sym(const ScaleSymJob* __restrict__ jobs) {
  const ScaleSymJob J = jobs[blockIdx.y];
  const long long total = (long long)J.q * J.q;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % J.q), j = (int)(e / J.q);
    J.G[i + j * J.ld] *= J.w[i] * J.w[j];
  }
}

__global__ void k_scale_rows(const ScaleRowsJob* __restrict__ jobs) {
  const ScaleRowsJob J = jobs[blockIdx.y];
  const long long total = (long long)J.rows * J.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % J.rows), j = (int)(e / J.rows);
    J.dst[i + j * J.ldd] = J.src[i + j * J.lds] * J.w[i];
  }
}

__global__ void k_gather(const GatherJob* __restrict__ jobs) {
  const GatherJob J = jobs[blockIdx.y];
  const long long total = (long long)J.rows * J.cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % J.rows), j = (int)(e / J.rows);
    const int sj = J.perm ? J.perm[j] : j;
    J.dst[i + j * J.ldd] = J.src[i + (long long)sj * J.lds];
  }
}

__global__ void k_colnorms2(const double* __restrict__ P, long long ld, int rows, int cols,
                            double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= cols) return;
  const double* col = P + (long long)c * ld;
  double acc = 0.0;
  for (int r = lane; r < rows; r += 32) acc += col[r] * col[r];
  acc = warp_sum(acc);
  if (lane == 0) out[c] = acc;
}

__global__ void k_ortho_defect(const double* G, long long ld, int q, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  const long long total = (long long)q * q;
  for (long long e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = (int)(e % q), j = (int)(e / q);
    const double v = G[i + j * ld] - (i == j ? 1.0 : 0.0);
    m = fmax(m, fabs(v));
    if (v != v) m = INFINITY;
  }
  m = block_max(m, red);
  if (threadIdx.x == 0) *out = m;
}

__global__ void k_transpose(const double* __restrict__ src, long long lds, int rows, int cols,
                            double* __restrict__ dst, long long ldd, int to_col) {
  // to_col: src row-major (rows x cols, lds) -> dst col-major (ldd)
  // else  : src col-major (lds)             -> dst row-major (ldd)
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  if (to_col) {
    // read rows of src coalesced along cols
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int r = by + k, c = bx + threadIdx.x;
      if (r < rows && c < cols) tile[k][threadIdx.x] = src[(long long)r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int c = bx + k, r = by + threadIdx.x;
      if (r < rows && c < cols) dst[r + (long long)c * ldd] = tile[threadIdx.x][k];
    }
  } else {
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int c = bx + k, r = by + threadIdx.x;
      if (r < rows && c < cols) tile[threadIdx.x][k] = src[r + (long long)c * lds];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
      const int r = by + k, c = bx + threadIdx.x;
      if (r < rows && c < cols) dst[(long long)r * ldd + c] = tile[k][threadIdx.x];
    }
  }
}

template <typename Job>
const Job* stage(Ctx& ctx, const std::vector<Job>& jobs) {
  return static_cast<const Job*>(ctx.staging.put(jobs.data(), jobs.size() * sizeof(Job), ctx.stream));
}

int grid_for(long long elems) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((elems + 255) / 256, 2048)));
}

}  // namespace

void finalize(Ctx& ctx, const std::vector<FinJob>& jobs) {
  if (jobs.empty()) return;
  int pmax = 0;
  for (auto& j : jobs) pmax = std::max(pmax, j.p);
  const size_t smem = (4 * (size_t)pmax + 32) * sizeof(double) + 2 * (size_t)pmax * sizeof(int) + 64;
  HSVD_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ctx.launch_begin();
  k_finalize<<<(unsigned)jobs.size(), FIN_THREADS, smem, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_finalize");
}

void scale_sym(Ctx& ctx, const std::vector<ScaleSymJob>& jobs) {
  if (jobs.empty()) return;
  long long mx = 0;
  for (auto& j : jobs) mx = std::max(mx, (long long)j.q * j.q);
  ctx.launch_begin();
  k_scale_sym<<<dim3(grid_for(mx), (unsigned)jobs.size()), 256, 0, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_scale_sym");
}

void scale_rows(Ctx& ctx, const std::vector<ScaleRowsJob>& jobs) {
  if (jobs.empty()) return;
  long long mx = 0;
  for (auto& j : jobs) mx = std::max(mx, (long long)j.rows * j.cols);
  ctx.launch_begin();
  k_scale_rows<<<dim3(grid_for(mx), (unsigned)jobs.size()), 256, 0, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_scale_rows");
}

void gather_cols(Ctx& ctx, const std::vector<GatherJob>& jobs) {
  if (jobs.empty()) return;
  long long mx = 0;
  for (auto& j : jobs) mx = std::max(mx, (long long)j.rows * j.cols);
  ctx.launch_begin();
  k_gather<<<dim3(grid_for(mx), (unsigned)jobs.size()), 256, 0, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_gather");
}

void colnorms2(Ctx& ctx, const double* P, long long ld, int rows, int cols, double* out) {
  if (cols <= 0) return;
  ctx.launch_begin();
  k_colnorms2<<<ceil_div(cols, 8), 256, 0, ctx.stream>>>(P, ld, rows, cols, out);
  ctx.check_launch("k_colnorms2");
}

void ortho_defect(Ctx& ctx, const double* G, long long ld, int q, double* out) {
  ctx.launch_begin();
  k_ortho_defect<<<1, 1024, 0, ctx.stream>>>(G, ld, q, out);
  ctx.check_launch("k_ortho_defect");
}

void rowmajor_to_colmajor(Ctx& ctx, const double* src, long long lds, int rows, int cols,
                          double* dst, long long ldd) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
  ctx.launch_begin();
  k_transpose<<<grid, dim3(32, 8), 0, ctx.stream>>>(src, lds, rows, cols, dst, ldd, 1);
  ctx.check_launch("k_transpose");
}

void colmajor_to_rowmajor(Ctx& ctx, const double* src, long long lds, int rows, int cols,
                          double* dst, long long ldd) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32));
  ctx.launch_begin();
  k_transpose<<<grid, dim3(32, 8), 0, ctx.stream>>>(src, lds, rows, cols, dst, ldd, 0);
  ctx.check_launch("k_transpose");
}

}  // namespace hsvdcu
