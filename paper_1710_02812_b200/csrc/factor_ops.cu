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
constexpr int NORM_CHUNK = 8192;  // rows per partial column norm

// Scratch of one finalisation (allocated by finalize()).
struct FinDev {
  FinJob j;
  double* part;   // nchunk x p partial squared norms
  int nchunk;
  double* scale;  // p: 1/sigma (1 for columns needing completion)
  int* info;      // [0] columns to write, [1] any column needs completion
};

// 1. partial squared column norms: block (chunk, column, job)
__global__ void k_colnorm_part(const FinDev* __restrict__ jobs) {
  const FinDev F = jobs[blockIdx.z];
  const int c = blockIdx.y, ch = blockIdx.x;
  if (c >= F.j.p || ch >= F.nchunk || F.j.norms2) return;
  const double* col = F.j.P + (long long)c * F.j.ldp;
  const int r0 = ch * NORM_CHUNK, r1 = min(F.j.s, r0 + NORM_CHUNK);
  double acc = 0.0;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc += col[r] * col[r];
  __shared__ double red[32];
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) F.part[(long long)ch * F.j.p + c] = acc;
}

// 3. U[:, i] = P[:, perm[i]] * scale[i] for the written columns
__global__ void k_scale_gather(const FinDev* __restrict__ jobs) {
  const FinDev F = jobs[blockIdx.z];
  const int i = blockIdx.y;
  if (i >= F.info[0]) return;
  const int src = F.j.perm[i];
  const double sc = F.scale[i];
  const double* in = F.j.P + (long long)src * F.j.ldp;
  double* out = F.j.U + (long long)i * F.j.ldu;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < F.j.s; r += gridDim.x * blockDim.x)
    out[r] = in[r] * sc;
}

// 2. sort, truncation count, scales (one CTA per job)
__global__ void __launch_bounds__(FIN_THREADS) k_finalize(const FinDev* __restrict__ jobs) {
  const FinDev F = jobs[blockIdx.x];
  const FinJob J = F.j;
  const int p = J.p;
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ double sm[];
  double* sig_old = sm;
  double* sig_new = sig_old + p;
  int* perm = reinterpret_cast<int*>(sig_new + p);
  __shared__ double s_smax;
  __shared__ int s_nan;
  if (tid == 0) s_nan = 0;
  for (int i = tid; i < p; i += nt) perm[i] = i;
  __syncthreads();
  for (int c = tid; c < p; c += nt) {
    double acc = 0.0;
    if (J.norms2) {
      acc = J.norms2[c];
    } else {
      for (int ch = 0; ch < F.nchunk; ++ch) acc += F.part[(long long)ch * p + c];
    }
    {
      double v = std::sqrt(acc);
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
    s_smax = smax;
    *J.rank = keep;
    *J.degenerate = deg;
    F.info[0] = J.write_all ? p : keep;
    F.info[1] = 0;
  }
  __syncthreads();
  const double smax = s_smax;
  const int wr = F.info[0];
  int anybad = 0;
  for (int i = tid; i < p; i += nt) {
    J.sigma[i] = sig_new[i];
    J.perm[i] = perm[i];
    const bool bad = !(sig_new[i] > 1e-6 * smax) || smax == 0.0;
    double inv = bad ? 1.0 : 1.0 / sig_new[i];
    // sharded: completion would need a global Gram-Schmidt (zero column instead)
    if (J.norms2) inv = sig_new[i] > 0.0 ? 1.0 / sig_new[i] : 0.0;
    F.scale[i] = inv;
    if (bad && i < wr && !J.norms2) anybad = 1;
  }
  if (anybad) atomicOr(&F.info[1], 1);
}

// 4. complete unstable / null directions in sigma order (rare: rank-deficient
// inputs; the kernel exits at once otherwise)
__global__ void __launch_bounds__(FIN_THREADS) k_complete(const FinDev* __restrict__ jobs) {
  const FinDev F = jobs[blockIdx.x];
  if (F.info[1] == 0) return;
  const FinJob J = F.j;
  const int s = J.s, p = J.p;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  extern __shared__ double sm[];
  double* dots = sm;
  double* red = dots + p;
  int* bad = reinterpret_cast<int*>(red + 32);
  const int wr = F.info[0];
  const double smax = J.sigma[0];
  for (int i = tid; i < p; i += nt) bad[i] = !(J.sigma[i] > 1e-6 * smax) || smax == 0.0;
  __syncthreads();
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

// C (k x k, SPD, ~identity) = R^T R; writes R^{-1} (upper) to Rinv.  One CTA;
// R kept in Rinv's storage during the factorisation, inverted in place by
// column-parallel back substitution into a scratch half.
__global__ void __launch_bounds__(1024) k_chol_inv(const double* __restrict__ C, int k,
                                                   double* __restrict__ R,
                                                   double* __restrict__ Rinv) {
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double s_d;
  __shared__ int s_bad;
  if (tid == 0) s_bad = 0;
  for (int e = tid; e < k * k; e += nt) R[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      double s = C[j + (long long)j * k];
      for (int i = 0; i < j; ++i) s -= R[i + j * k] * R[i + j * k];
      if (!(s > 0.0)) {
        s_bad = 1;
        s = 1.0;
      }
      s_d = sqrt(s);
      R[j + j * k] = s_d;
    }
    __syncthreads();
    const double djj = s_d;
    for (int l = j + 1 + tid; l < k; l += nt) {
      double s = C[j + (long long)l * k];
      for (int i = 0; i < j; ++i) s -= R[i + j * k] * R[i + l * k];
      R[j + l * k] = s / djj;
    }
    __syncthreads();
  }
  // R^{-1}: column c solves R x = e_c
  for (int c = tid; c < k; c += nt) {
    for (int i = 0; i < k; ++i) Rinv[i + c * k] = 0.0;
    for (int i = c; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int l = i + 1; l <= c; ++l) s -= R[i + l * k] * Rinv[l + c * k];
      Rinv[i + c * k] = s / R[i + i * k];
    }
  }
  __syncthreads();
  if (s_bad)  // not positive definite (cannot happen for a near-orthonormal U): identity
    for (int e = tid; e < k * k; e += nt) Rinv[e] = (e % k == e / k) ? 1.0 : 0.0;
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
  int pmax = 0, chmax = 1, smax = 1;
  // algorithmic HBM bytes (profile): the norms read P once; the gather reads
  // and writes the written columns (min(p, cap), all p with write_all)
  double norm_bytes = 0.0, gather_bytes = 0.0;
  std::vector<FinDev> dev(jobs.size());
  for (size_t i = 0; i < jobs.size(); ++i) {
    FinDev& f = dev[i];
    f.j = jobs[i];
    if (!f.j.perm) f.j.perm = ctx.arena.alloc_n<int>(f.j.p);
    f.nchunk = std::max(1, ceil_div(f.j.s, NORM_CHUNK));
    f.part = ctx.arena.alloc_n<double>((size_t)f.nchunk * f.j.p);
    f.scale = ctx.arena.alloc_n<double>(f.j.p);
    f.info = ctx.arena.alloc_n<int>(2);
    pmax = std::max(pmax, f.j.p);
    chmax = std::max(chmax, f.nchunk);
    smax = std::max(smax, f.j.s);
    if (!f.j.norms2) norm_bytes += 8.0 * f.j.s * f.j.p;
    gather_bytes += 16.0 * f.j.s * ((f.j.write_all || f.j.cap <= 0) ? f.j.p : std::min(f.j.p, f.j.cap));
  }
  const FinDev* dd = stage(ctx, dev);
  const unsigned nj = (unsigned)dev.size();
  ctx.launch_begin();
  ctx.pending_bytes = norm_bytes;
  k_colnorm_part<<<dim3(chmax, pmax, nj), 256, 0, ctx.stream>>>(dd);
  ctx.check_launch("k_colnorm_part");
  const size_t smem = 2 * (size_t)pmax * sizeof(double) + (size_t)pmax * sizeof(int) + 64;
  smem_optin(k_finalize, smem);
  ctx.launch_begin();
  k_finalize<<<nj, FIN_THREADS, smem, ctx.stream>>>(dd);
  ctx.check_launch("k_finalize");
  const int gx = std::min(ceil_div(smax, 256 * 4), 64);
  ctx.launch_begin();
  ctx.pending_bytes = gather_bytes;
  k_scale_gather<<<dim3(gx, pmax, nj), 256, 0, ctx.stream>>>(dd);
  ctx.check_launch("k_scale_gather");
  const size_t smem2 = ((size_t)pmax + 32) * sizeof(double) + (size_t)pmax * sizeof(int) + 64;
  smem_optin(k_complete, smem2);
  ctx.launch_begin();
  k_complete<<<nj, FIN_THREADS, smem2, ctx.stream>>>(dd);
  ctx.check_launch("k_complete");
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
  double bytes = 0.0;
  for (auto& j : jobs) {
    mx = std::max(mx, (long long)j.rows * j.cols);
    bytes += 16.0 * j.rows * j.cols;
  }
  ctx.launch_begin();
  ctx.pending_bytes = bytes;
  k_scale_rows<<<dim3(grid_for(mx), (unsigned)jobs.size()), 256, 0, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_scale_rows");
}

void gather_cols(Ctx& ctx, const std::vector<GatherJob>& jobs) {
  if (jobs.empty()) return;
  long long mx = 0;
  double bytes = 0.0;
  for (auto& j : jobs) {
    mx = std::max(mx, (long long)j.rows * j.cols);
    bytes += 16.0 * j.rows * j.cols;
  }
  ctx.launch_begin();
  ctx.pending_bytes = bytes;
  k_gather<<<dim3(grid_for(mx), (unsigned)jobs.size()), 256, 0, ctx.stream>>>(stage(ctx, jobs));
  ctx.check_launch("k_gather");
}

void chol_inverse(Ctx& ctx, const double* C, int k, double* Rinv) {
  double* R = ctx.arena.alloc_n<double>((size_t)k * k);
  ctx.launch_begin();
  k_chol_inv<<<1, 1024, 0, ctx.stream>>>(C, k, R, Rinv);
  ctx.check_launch("k_chol_inv");
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
