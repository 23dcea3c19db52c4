// One-sided (Hestenes) Jacobi SVD of narrow matrices on the device: the
// reference's route for every SVD whose smaller side is <= 32
// (kernels.cpp:28: JacobiSVD when min(rows, cols) <= 32).
//
// The Gram route every other SVD of the path takes (eigenpairs of A^T A, then
// P = A Z) loses relative accuracy on small singular values (error
// eps * kappa^2); rotating the columns of A itself keeps it at eps * kappa
// (and small singular values to high relative accuracy), which is what the
// reference's own pins assume (tests/test_factor.cpp:176-198: rank_k_error
// 8.1960876183812958e-09 to 1e-6).  The outputs are exactly what the Gram
// route hands to finalize: P = A V (s x w, columns = U sigma) and V (w x w),
// columns ordered by decreasing norm.
//
// One CTA per matrix: the columns live in a column-major scratch copy; each
// sweep is w-1 rounds of the round-robin (circle) pairing, every warp rotates
// one disjoint column pair per round (3 dot products + the rotation, fixed
// reduction order: bitwise deterministic), V in shared memory.  Converged
// when no pair has |a_p . a_q| > sqrt(s) eps |a_p| |a_q| (LAPACK dgesvj's
// tolerance).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "jacobi.h"

namespace hsvdcu {

namespace {

constexpr int kJacThreads = 512;  // 16 warps: one per pair of a 32-column round
constexpr int kMaxSweeps = 60;

__global__ void __launch_bounds__(kJacThreads) k_jacobi(const JacJob* __restrict__ jobs) {
  __shared__ double Vs[kJacMaxW][kJacMaxW + 1];  // V[i][j]
  __shared__ double nrm[kJacMaxW];
  __shared__ int perm[kJacMaxW];
  __shared__ int rotated;
  const JacJob J = jobs[blockIdx.x];
  const int w = J.w1 + J.w2;
  const long long s = J.s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* W = J.W;
  for (long long e = tid; e < s * w; e += kJacThreads) {
    const int j = static_cast<int>(e % w);
    const long long i = e / w;
    double v;
    if (j < J.w1) {
      const long long off = i * J.rs + (long long)j * J.cs;
      v = J.f64 ? static_cast<const double*>(J.A)[off]
                : static_cast<double>(static_cast<const float*>(J.A)[off]);
      if (J.s1) v *= J.s1[j];
    } else {
      const int jj = j - J.w1;
      v = J.A2[i + (long long)jj * J.ld2];
      if (J.s2) v *= J.s2[jj];
    }
    W[i + (long long)j * s] = v;
  }
  for (int e = tid; e < kJacMaxW * kJacMaxW; e += kJacThreads)
    Vs[e / kJacMaxW][e % kJacMaxW] = (e / kJacMaxW == e % kJacMaxW) ? 1.0 : 0.0;
  const double tol = sqrt((double)s) * 2.220446049250313e-16;
  const int wp = w + (w & 1);  // odd w: one dummy player
  __syncthreads();
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < wp - 1; ++r) {
      if (warp < wp / 2) {
        auto at = [&](int m) { return m == 0 ? 0 : 1 + (m - 1 + r) % (wp - 1); };
        int p = at(warp), q = at(wp - 1 - warp);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        if (q < w) {
          double* cp = W + (long long)p * s;
          double* cq = W + (long long)q * s;
          double a = 0.0, b = 0.0, g = 0.0;
          for (long long i = lane; i < s; i += 32) {
            const double x = cp[i], y = cq[i];
            a += x * x;
            b += y * y;
            g += x * y;
          }
          a = warp_sum(a);
          b = warp_sum(b);
          g = warp_sum(g);
          if (g != 0.0 && fabs(g) > tol * sqrt(a) * sqrt(b)) {
            const double zeta = (b - a) / (2.0 * g);
            const double t = fabs(zeta) > 1e150
                                 ? 0.5 / zeta
                                 : copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
            for (long long i = lane; i < s; i += 32) {
              const double x = cp[i], y = cq[i];
              cp[i] = c * x - sn * y;
              cq[i] = sn * x + c * y;
            }
            if (lane < w) {
              const double x = Vs[lane][p], y = Vs[lane][q];
              Vs[lane][p] = c * x - sn * y;
              Vs[lane][q] = sn * x + c * y;
            }
            if (lane == 0) rotated = 1;
          }
        }
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) break;
  }
  // column norms, order by decreasing norm (stable), write P and V
  for (int j = warp; j < w; j += kJacThreads / 32) {
    const double* cj = W + (long long)j * s;
    double a = 0.0;
    for (long long i = lane; i < s; i += 32) a += cj[i] * cj[i];
    a = warp_sum(a);
    if (lane == 0) nrm[j] = sqrt(a);
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < w; ++j) perm[j] = j;
    for (int j = 1; j < w; ++j) {  // insertion sort, descending, stable
      const int pj = perm[j];
      int k = j - 1;
      while (k >= 0 && nrm[perm[k]] < nrm[pj]) {
        perm[k + 1] = perm[k];
        --k;
      }
      perm[k + 1] = pj;
    }
  }
  __syncthreads();
  for (long long e = tid; e < s * w; e += kJacThreads) {
    const int c = static_cast<int>(e / s);
    const long long i = e % s;
    J.P[i + (long long)c * J.ldp] = W[i + (long long)perm[c] * s];
  }
  for (int e = tid; e < w * w; e += kJacThreads) {
    const int c = e / w, i = e % w;
    J.Z[i + (long long)c * J.ldz] = Vs[i][perm[c]];
  }
}

// ---------------------------------------------------------------------------
// Householder thin QR (kernels.cpp:50-61 qr_thin: Eigen HouseholderQR, thin Q
// = householderQ() * I).  LAPACK dgeqrf/dorg2r conventions (beta =
// -sign(alpha) ||x||, the sign Eigen's makeHouseholder uses too).  One CTA per
// matrix: per column a block reduction forms the reflector, then the warps
// update the trailing columns (one column per warp, fixed reduction order);
// Q is accumulated backwards from the identity.  A building block exported
// for the reference's API (the merges run in Gram/Jacobi form and do not
// call it).
// ---------------------------------------------------------------------------
constexpr int kQrThreads = 512;

__global__ void __launch_bounds__(kQrThreads) k_householder_qr(double* __restrict__ A, int m,
                                                               int n, double* __restrict__ tau,
                                                               double* __restrict__ Q) {
  __shared__ double red[kQrThreads / 32];
  __shared__ double sh_beta, sh_tau, sh_scal;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = kQrThreads / 32;
  const int p = min(m, n);
  auto col = [&](double* B, int c) { return B + (long long)c * m; };
  for (int j = 0; j < p; ++j) {
    double* aj = col(A, j);
    double x2 = 0.0;
    for (int i = j + 1 + tid; i < m; i += kQrThreads) x2 += aj[i] * aj[i];
    x2 = block_sum(x2, red);
    if (tid == 0) {
      const double alpha = aj[j];
      if (x2 == 0.0) {
        sh_tau = 0.0;
        sh_beta = alpha;
        sh_scal = 0.0;
      } else {
        const double beta = -copysign(sqrt(alpha * alpha + x2), alpha);
        sh_tau = (beta - alpha) / beta;
        sh_scal = 1.0 / (alpha - beta);
        sh_beta = beta;
      }
    }
    __syncthreads();
    const double t = sh_tau, sc = sh_scal;
    for (int i = j + 1 + tid; i < m; i += kQrThreads) aj[i] *= sc;  // v below the diagonal
    __syncthreads();
    if (tid == 0) {
      aj[j] = sh_beta;
      tau[j] = t;
    }
    if (t != 0.0) {
      for (int c = j + 1 + warp; c < n; c += nw) {
        double* ac = col(A, c);
        double w = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w += aj[i] * ac[i];
        w = warp_sum(w) + ac[j];
        w *= t;
        for (int i = j + 1 + lane; i < m; i += 32) ac[i] -= w * aj[i];
        if (lane == 0) ac[j] -= w;
      }
    }
    __syncthreads();
  }
  // Q (m x p) = H_0 ... H_{p-1} I, accumulated backwards
  for (long long e = tid; e < (long long)m * p; e += kQrThreads)
    Q[e] = (e % m == e / m) ? 1.0 : 0.0;
  __syncthreads();
  for (int j = p - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t != 0.0) {
      const double* v = col(A, j);
      for (int c = j + warp; c < p; c += nw) {
        double* qc = col(Q, c);
        double w = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w += v[i] * qc[i];
        w = warp_sum(w) + qc[j];
        w *= t;
        for (int i = j + 1 + lane; i < m; i += 32) qc[i] -= w * v[i];
        if (lane == 0) qc[j] -= w;
      }
    }
    __syncthreads();
  }
}

}  // namespace

void householder_qr(Ctx& ctx, double* A, int m, int n, double* Q) {
  double* tau = ctx.arena.alloc_n<double>(std::max(1, std::min(m, n)));
  ctx.launch_begin();
  k_householder_qr<<<1, kQrThreads, 0, ctx.stream>>>(A, m, n, tau, Q);
  ctx.check_launch("k_householder_qr");
}

bool small_svd_jacobi(long long s, int w) {
  if (w < 1 || w > kJacMaxW || s > (1LL << 20)) return false;
  const char* e = std::getenv("HSVD_SMALL_SVD");
  return !(e && std::strcmp(e, "gram") == 0);
}

void jacobi_svd_batch(Ctx& ctx, std::vector<JacJob>& jobs) {
  if (jobs.empty()) return;
  for (auto& j : jobs) {
    const int w = j.w1 + j.w2;
    if (w < 1 || w > kJacMaxW) throw Error(kInvalid, "jacobi_svd_batch: width out of range");
    if (!j.W) j.W = ctx.arena.alloc_n<double>((size_t)j.s * w);
  }
  const JacJob* dj = static_cast<const JacJob*>(ctx.staging.put_to(
      ctx.arena.alloc(jobs.size() * sizeof(JacJob)), jobs.data(), jobs.size() * sizeof(JacJob),
      ctx.stream));
  ctx.launch_begin();
  k_jacobi<<<(unsigned)jobs.size(), kJacThreads, 0, ctx.stream>>>(dj);
  ctx.check_launch("k_jacobi");
}

}  // namespace hsvdcu
