// Batched fp64 symmetric eigensolver, top-kk eigenpairs (one matrix per CTA
// for the latency-bound phases, grouped DMMA GEMMs for the back-transform).
//
// Replaces the dense SVD kernel of the reference (Eigen BDCSVD/JacobiSVD,
// kernels.cpp:21-48) on the Gram form of every decomposition in the path:
// a block X_b (d x c) is decomposed through G = X_b^T X_b (c x c), whose top
// eigenpairs give (sigma^2, V_b); U_b = X_b V_b / sigma follows by GEMM.
//
//   1. k_sytrd   Householder tridiagonalisation Q^T G Q = T (LAPACK dsytd2 'L'
//                algorithm), with the rank-2 update of step j fused with the
//                symmetric mat-vec of step j+1: one read+write pass of the
//                trailing matrix per column.
//   2. k_steig   top-kk eigenvalues of T by Sturm-count bisection, vectors by
//                LDL^T inverse iteration with Gram-Schmidt inside clusters
//                (LAPACK dstebz + dstein algorithm).
//   3. back-transform Z <- Q Z with the compact-WY form of 32 reflectors at a
//                time (LAPACK dlarft + dlarfb): three grouped DMMA GEMMs per
//                reflector block, the reflectors read in place from A.
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "gemm.h"
#include "syev.h"

namespace cg = cooperative_groups;

namespace hsvdcu {

namespace {

constexpr int TRD_THREADS = 1024;
constexpr int TRD_QMAX = 8;  // rows per thread when n > 1024 (n <= 8192)
constexpr int EIG_THREADS = 512;
constexpr int NB = 32;       // reflectors per compact-WY block
constexpr int B2 = 32;       // bandwidth of the two-stage reduction
constexpr int LDBB = 2 * B2 + 1;  // band storage: diagonals 0..2*B2 (chase fill)
constexpr int kBandInvitMinN = 1 << 30;  // band inverse iteration: only when forced
constexpr int kBandGroupDefault = 4;  // panels per delayed trailing update (two-stage stage 1)
constexpr int INV_WARPS = 4;      // warps (= LU workspace slots) per band inverse iteration CTA

struct EigDev {
  double* A;
  long long lda;
  int n;
  int kk;
  double* d;
  double* e;
  double* tau;
  double* lam;
  double* Z;
  long long ldz;
  double* piv;   // n * kk scratch (LDL^T pivots)
  double* T;     // (nblocks * NBT * NBT) compact-WY T factors
  double* S;     // (nblocks * NBT * NBT) V^T V of each reflector block
  double* VW;    // n x 2*NB panel [V | W] (blocked tridiagonalisation)
  double* WV;    // n x 2*NB panel [W | V]
  // two-stage path
  int vals_only;     // k_steig: 1 eigenvalues (+ shifts, clusters) only; 2 vectors
                     // without the in-iteration Gram-Schmidt (k_band_mgs follows)
  double* shifts;    // kk perturbed inverse-iteration shifts
  int* cstarts;      // kk cluster starts
  double* band;      // (2*B2+1) x n lower band, chased to tridiagonal
  double* band0;     // copy of the band after stage 1 (inverse iteration)
  double* Tp;        // npanels x B2 x B2 panel T factors
  double* psum;      // 8 x B2 x B2 per-CTA partials of V^T V (k_panel_qr)
  double* Y;         // n x B2
  double* P1;        // B2 x B2
  double* Mb;        // B2 x B2
  double* Z1;        // (2*B2*group) x B2: pending-update products
  double* lu;        // per-warp band LU workspace (cpm * INV_WARPS slots per matrix)
  double* refl;      // chase reflectors: (steps) x 33 (v[0..31], tau), sweep-major
  long long lu_slot;  // doubles per slot
};

// ---------------------------------------------------------------------------
// 1. tridiagonalisation
// ---------------------------------------------------------------------------

// Householder reflector (LAPACK dlarfg) annihilating A[r0+1:, c]; v has
// v[r0] = 1, stored to vout[r0..n) and to A[r0+1:, c].  Returns tau.
__device__ double make_reflector(double* A, long long lda, int n, int c, int r0, double* vout,
                                 double* red, double* e_out, double* tau_out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double part = 0.0;
  for (int i = r0 + 1 + tid; i < n; i += nt) {
    const double x = A[i + c * lda];
    part += x * x;
  }
  const double xn2 = block_sum(part, red);
  const double alpha = A[r0 + c * lda];
  double tau = 0.0, beta = alpha, scal = 0.0;
  if (xn2 > 0.0) {
    const double nrm = sqrt(alpha * alpha + xn2);
    beta = alpha >= 0.0 ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  for (int i = r0 + 1 + tid; i < n; i += nt) {
    const double v = A[i + c * lda] * scal;
    A[i + c * lda] = v;
    vout[i] = v;
  }
  if (tid == 0) {
    vout[r0] = 1.0;
    *e_out = beta;
    *tau_out = tau;
  }
  return tau;
}

// One pass over the trailing block A[lo:, lo:]: optional rank-2 update
// A -= v w^T + w v^T, and p = A_new * mv.  p written to ps[lo..n).
template <bool UPDATE>
__device__ void trailing_pass(double* A, long long lda, int n, int lo, const double* vs,
                              const double* wv, const double* mv, double* ps, double* pp,
                              int RT, int CT, int tr, int tc) {
  double pacc[TRD_QMAX];
  double vi[TRD_QMAX], wi[TRD_QMAX];
  int Q = (n - lo + RT - 1) / RT;
  if (Q > TRD_QMAX) Q = TRD_QMAX;
#pragma unroll
  for (int q = 0; q < TRD_QMAX; ++q) {
    pacc[q] = 0.0;
    const int i = lo + tr + q * RT;
    vi[q] = (q < Q && i < n && UPDATE) ? vs[i] : 0.0;
    wi[q] = (q < Q && i < n && UPDATE) ? wv[i] : 0.0;
  }
  int k = lo + tc;
  // unrolled by 2 columns for memory-level parallelism
  for (; k + CT < n; k += 2 * CT) {
    const int k1 = k + CT;
    const double mk0 = mv[k], mk1 = mv[k1];
    double vk0 = 0, wk0 = 0, vk1 = 0, wk1 = 0;
    if (UPDATE) {
      vk0 = vs[k]; wk0 = wv[k]; vk1 = vs[k1]; wk1 = wv[k1];
    }
    double* c0 = A + (long long)k * lda;
    double* c1 = A + (long long)k1 * lda;
#pragma unroll
    for (int q = 0; q < TRD_QMAX; ++q) {
      const int i = lo + tr + q * RT;
      if (q < Q && i < n) {
        double a0 = c0[i], a1 = c1[i];
        if (UPDATE) {
          a0 -= vi[q] * wk0 + wi[q] * vk0;
          a1 -= vi[q] * wk1 + wi[q] * vk1;
          c0[i] = a0;
          c1[i] = a1;
        }
        pacc[q] += a0 * mk0 + a1 * mk1;
      }
    }
  }
  for (; k < n; k += CT) {
    const double mk = mv[k];
    double vk = 0, wk = 0;
    if (UPDATE) { vk = vs[k]; wk = wv[k]; }
    double* c0 = A + (long long)k * lda;
#pragma unroll
    for (int q = 0; q < TRD_QMAX; ++q) {
      const int i = lo + tr + q * RT;
      if (q < Q && i < n) {
        double a = c0[i];
        if (UPDATE) {
          a -= vi[q] * wk + wi[q] * vk;
          c0[i] = a;
        }
        pacc[q] += a * mk;
      }
    }
  }
  if (CT == 1) {
#pragma unroll
    for (int q = 0; q < TRD_QMAX; ++q) {
      const int i = lo + tr + q * RT;
      if (q < Q && i < n) ps[i] = pacc[q];
    }
  } else {
    pp[tc * RT + tr] = pacc[0];  // Q == 1 whenever CT > 1
    __syncthreads();
    if (threadIdx.x < RT) {
      const int i = lo + threadIdx.x;
      double s = 0.0;
      for (int c = 0; c < CT; ++c) s += pp[c * RT + threadIdx.x];
      if (i < n) ps[i] = s;
    }
  }
}

__global__ void __launch_bounds__(TRD_THREADS) k_sytrd(const EigDev* __restrict__ jobs) {
  const EigDev J = jobs[blockIdx.x];
  const int n = J.n;
  double* A = J.A;
  const long long lda = J.lda;
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ double sm[];
  double* vs = sm;
  double* wv = vs + n;
  double* vn = wv + n;
  double* ps = vn + n;
  double* pp = ps + n;
  double* red = pp + TRD_THREADS;
  __shared__ double s_tau, s_tau_next, s_e;

  if (n == 1) {
    if (tid == 0) J.d[0] = A[0];
    return;
  }
  int RT = 32;
  while (RT < n && RT < TRD_THREADS) RT <<= 1;
  const int CT = nt / RT;
  const int tr = tid % RT, tc = tid / RT;

  // reflector 0 from column 0
  make_reflector(A, lda, n, 0, 1, vn, red, &s_e, &s_tau);
  __syncthreads();
  if (tid == 0) {
    J.d[0] = A[0];
    J.e[0] = s_e;
    J.tau[0] = s_tau;
  }
  for (int i = 1 + tid; i < n; i += nt) vs[i] = vn[i];
  __syncthreads();
  trailing_pass<false>(A, lda, n, 1, vs, wv, vs, ps, pp, RT, CT, tr, tc);
  __syncthreads();

  for (int j = 0; j <= n - 2; ++j) {
    const double tau = s_tau;
    if (tau != 0.0) {
      double part = 0.0;
      for (int i = j + 1 + tid; i < n; i += nt) part += ps[i] * vs[i];
      const double dot = tau * block_sum(part, red);
      const double alpha = -0.5 * tau * dot;
      for (int i = j + 1 + tid; i < n; i += nt) wv[i] = tau * ps[i] + alpha * vs[i];
    } else {
      for (int i = j + 1 + tid; i < n; i += nt) wv[i] = 0.0;
    }
    __syncthreads();
    if (j == n - 2) {
      if (tid == 0) {
        const long long ii = (long long)(n - 1) * (lda + 1);
        J.d[n - 1] = A[ii] - 2.0 * vs[n - 1] * wv[n - 1];
      }
      break;
    }
    // update column j+1 (rows j+1..n-1)
    {
      const long long cj = (long long)(j + 1) * lda;
      const double vj = vs[j + 1], wj = wv[j + 1];
      for (int i = j + 1 + tid; i < n; i += nt) A[i + cj] -= vs[i] * wj + wv[i] * vj;
    }
    __syncthreads();
    make_reflector(A, lda, n, j + 1, j + 2, vn, red, &s_e, &s_tau_next);
    __syncthreads();
    if (tid == 0) {
      J.d[j + 1] = A[(long long)(j + 1) * (lda + 1)];
      J.e[j + 1] = s_e;
      J.tau[j + 1] = s_tau_next;
    }
    trailing_pass<true>(A, lda, n, j + 2, vs, wv, vn, ps, pp, RT, CT, tr, tc);
    __syncthreads();
    for (int i = j + 2 + tid; i < n; i += nt) vs[i] = vn[i];
    if (tid == 0) s_tau = s_tau_next;
    __syncthreads();
  }
}

// Blocked tridiagonalisation (LAPACK dlatrd 'L' algorithm): one launch per
// panel of NB columns.  Per column: update it with the panel's earlier
// (v, w) pairs, form the reflector, and compute w = tau*(A22 v - V(W^T v) -
// W(V^T v)) - ... with A22 read-only (its panel-start value).  The trailing
// rank-2*NB update A22 -= V W^T + W V^T follows as one symmetric DMMA GEMM.
// Thread i owns rows i, i+LAT, i+2*LAT, ... (coalesced column reads).
//
// Multi-SM: a cluster of CS CTAs shares one matrix.  Every CTA redundantly
// does the O(n*NB) per-column work (column update, reflector, corrections);
// the O(n^2) mat-vec is split by columns, each CTA streaming 1/CS of A22, and
// the CS partial vectors are exchanged through distributed shared memory and
// summed in rank order (bitwise identical in every CTA, deterministic).
constexpr int LAT = 512;

template <int R>
__global__ void __launch_bounds__(LAT, 1) k_latrd(const EigDev* __restrict__ jobs, int j0, int CS) {
  const EigDev J = jobs[blockIdx.x / CS];
  const int crank = blockIdx.x % CS;
  const int n = J.n;
  const int nref = n - 1;
  if (j0 >= nref || n <= 2) return;
  const int nbp = min(NB, nref - j0);
  double* A = J.A;
  const long long lda = J.lda;
  const double* VW = J.VW;
  const long long ldp = n;  // panel arrays are n x 2NB, ld n
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = LAT >> 5;
  extern __shared__ double sm[];
  double* vs = sm;                 // v by global row
  double* vrow = vs + n;           // V[j, 0:t], W[j, 0:t]
  double* c12 = vrow + 2 * NB;     // W^T v, V^T v
  double* red = c12 + 2 * NB;
  double* recv = red + 32;         // [2][CS][n] partial mat-vecs (double-buffered)
  __shared__ double s_alpha, s_diag;
  cg::cluster_group cluster = cg::this_cluster();
  // every CTA of the cluster must be running before its shared memory is
  // written by a peer (the early return above is uniform over the cluster)
  if (CS > 1) cluster.sync();

  for (int t = 0; t < nbp; ++t) {
    const int j = j0 + t;
    if (tid < t) {
      vrow[tid] = VW[j + (long long)tid * ldp];
      vrow[NB + tid] = VW[j + (long long)(NB + tid) * ldp];
    }
    __syncthreads();
    // (b) column j with the panel corrections
    double a[R];
    double part = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = tid + q * LAT;
      a[q] = 0.0;
      if (i >= j && i < n) {
        double s = A[i + (long long)j * lda];
        for (int u = 0; u < t; ++u)
          s -= VW[i + (long long)u * ldp] * vrow[NB + u] + VW[i + (long long)(NB + u) * ldp] * vrow[u];
        a[q] = s;
        if (i == j) s_diag = s;
        if (i == j + 1) s_alpha = s;
        if (i >= j + 2) part += s * s;
      }
    }
    const double xn2 = block_sum(part, red);
    const double alpha = s_alpha;
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      const double nrm = sqrt(alpha * alpha + xn2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (tid == 0) {
      J.d[j] = s_diag;
      J.e[j] = beta;
      J.tau[j] = tau;
    }
    double* Vt = J.VW + (long long)t * ldp;
    double* Vt2 = J.WV + (long long)(NB + t) * ldp;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = tid + q * LAT;
      if (i >= j + 1 && i < n) {
        const double v = (i == j + 1) ? 1.0 : a[q] * scal;
        vs[i] = v;
        Vt[i] = v;
        Vt2[i] = v;
      }
    }
    __syncthreads();
    // (d) p = A22 v (A22 = A[j+1:, j+1:], read-only); this CTA's columns only
    double p[R];
#pragma unroll
    for (int q = 0; q < R; ++q) p[q] = 0.0;
    int qlo = 0;
    while (qlo < R && tid + qlo * LAT < j + 1) ++qlo;
    const int chunk = (n - j - 1 + CS - 1) / CS;
    const int kb = j + 1 + crank * chunk;
    const int ke = min(n, kb + chunk);
    if (tau != 0.0 && qlo < R && kb < ke) {
      // Rows outside [j+1, n) read a clamped valid row and are discarded, so
      // the inner loop is branch-free and all U*R loads issue back to back.
      int ic[R];
#pragma unroll
      for (int q = 0; q < R; ++q) ic[q] = min(max(tid + q * LAT, j + 1), n - 1);
      constexpr int U = (R <= 3) ? 8 : (R <= 6 ? 6 : 3);
      int k = kb;
      for (; k + U <= ke; k += U) {
        const double* c0 = A + (long long)k * lda;
        double x[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < R; ++q) x[u][q] = __ldg(c0 + (long long)u * lda + ic[q]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const double vk = vs[k + u];
#pragma unroll
          for (int q = 0; q < R; ++q) p[q] = fma(x[u][q], vk, p[q]);
        }
      }
      for (; k < ke; ++k) {
        const double vk = vs[k];
        const double* c0 = A + (long long)k * lda;
#pragma unroll
        for (int q = 0; q < R; ++q) p[q] = fma(__ldg(c0 + ic[q]), vk, p[q]);
      }
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (q < qlo || tid + q * LAT >= n) p[q] = 0.0;
    }
    if (CS > 1) {  // exchange the partial mat-vecs through DSMEM
      double* buf = recv + (size_t)(t & 1) * CS * n;
      for (int rr = 0; rr < CS; ++rr) {
        double* peer = cluster.map_shared_rank(buf, rr);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const int i = tid + q * LAT;
          if (q >= qlo && i < n) peer[crank * n + i] = p[q];
        }
      }
      cluster.sync();
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = tid + q * LAT;
        if (q >= qlo && i < n) {
          double s = 0.0;
          for (int rr = 0; rr < CS; ++rr) s += buf[rr * n + i];
          p[q] = s;
        }
      }
    }
    // reflector storage (after the exchange: no CTA still reads column j)
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = tid + q * LAT;
      if (i >= j + 2 && i < n) A[i + (long long)j * lda] = vs[i];
    }
    // (e) panel corrections: p -= V (W^T v) + W (V^T v)
    if (t > 0 && tau != 0.0) {
      for (int u = warp; u < 2 * t; u += nwarps) {
        const double* col = J.VW + (long long)(u < t ? NB + u : u - t) * ldp;
        double s = 0.0;
        for (int i = j + 1 + lane; i < n; i += 32) s += col[i] * vs[i];
        s = warp_sum(s);
        if (lane == 0) c12[u] = s;  // c12[0:t] = W^T v, c12[t:2t] = V^T v
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int i = tid + q * LAT;
        if (q >= qlo && i < n) {
          double s = p[q];
          for (int u = 0; u < t; ++u)
            s -= VW[i + (long long)u * ldp] * c12[u] + VW[i + (long long)(NB + u) * ldp] * c12[t + u];
          p[q] = s;
        }
      }
    }
    // (f) w = tau p - 1/2 tau^2 (p.v) v
    double dp = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = tid + q * LAT;
      if (q >= qlo && i < n) dp += p[q] * vs[i];
    }
    const double dot = tau * block_sum(dp, red);
    const double al = -0.5 * tau * dot;
    double* Wt = J.VW + (long long)(NB + t) * ldp;
    double* Wt2 = J.WV + (long long)t * ldp;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int i = tid + q * LAT;
      if (i >= j + 1 && i < n) {
        const double w = tau * p[q] + al * vs[i];
        Wt[i] = w;
        Wt2[i] = w;
      }
    }
    __syncthreads();
  }
  if (j0 + nbp == nref && tid == 0) {
    const int i = n - 1;
    double s = A[(long long)i * (lda + 1)];
    for (int u = 0; u < nbp; ++u)
      s -= 2.0 * VW[i + (long long)u * ldp] * VW[i + (long long)(NB + u) * ldp];
    J.d[n - 1] = s;
  }
}

// ---------------------------------------------------------------------------
// 2. tridiagonal eigenpairs: bisection + inverse iteration
// ---------------------------------------------------------------------------

__device__ __forceinline__ int sturm_count_less(const double* dd, const double* e2, int n,
                                                double x, double pivmin) {
  double q = dd[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int cnt = q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = dd[i] - x - e2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

__device__ __forceinline__ double guard_pivot(double D, double tiny) {
  if (fabs(D) < tiny) return D < 0.0 ? -tiny : tiny;
  return D;
}

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void __launch_bounds__(EIG_THREADS) k_steig(const EigDev* __restrict__ jobs) {
  const EigDev J = jobs[blockIdx.x];
  const int n = J.n, kk = J.kk;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  extern __shared__ double sm[];
  double* dd = sm;
  double* ee = dd + n;
  double* e2 = ee + n;
  double* lam = e2 + n;
  double* shift = lam + kk;
  double* dots = shift + kk;
  double* red = dots + kk;
  int* cstart = reinterpret_cast<int*>(red + 32);

  double lo_g = 1e308, hi_g = -1e308, ee2max = 0.0;
  for (int i = tid; i < n; i += nt) {
    const double di = J.d[i];
    const double ei = i < n - 1 ? J.e[i] : 0.0;
    const double eim = i > 0 ? J.e[i - 1] : 0.0;
    dd[i] = di;
    ee[i] = ei;
    e2[i] = ei * ei;
    const double r = fabs(ei) + fabs(eim);
    lo_g = fmin(lo_g, di - r);
    hi_g = fmax(hi_g, di + r);
    ee2max = fmax(ee2max, ei * ei);
  }
  const double gl = -block_max(-lo_g, red);
  const double gu = block_max(hi_g, red);
  const double e2m = block_max(ee2max, red);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  const double eps = DBL_EPSILON;

  if (!(tnorm > 0.0) || !isfinite(tnorm)) {
    // zero (or non-finite) matrix: eigenvalues 0, vectors = identity columns
    for (int t = tid; t < kk; t += nt) {
      J.lam[t] = isfinite(tnorm) ? 0.0 : tnorm;
      double* z = J.Z + (long long)t * J.ldz;
      for (int r = 0; r < n; ++r) z[r] = (r == t) ? 1.0 : 0.0;
    }
    return;
  }
  const double pivmin = DBL_MIN * fmax(1.0, e2m);

  // eigenvalue with ascending index n-1-t (dstebz's tolerance): multisection
  // with P = nt / kk threads per eigenvalue -- each round evaluates P
  // interior points of the bracket and keeps the sub-interval holding the
  // eigenvalue (P = 1 is bisection), so the sequential Sturm counts per
  // eigenvalue drop from ~52 to ~52 / log2(P + 1)
  {
    const int P = max(1, nt / kk);
    double* blo = dots;  // [kk] bracket (the dots scratch is free here)
    double* bhi = shift;
    int* cnt = reinterpret_cast<int*>(cstart);  // [kk * P] (cstart is set later)
    for (int t = tid; t < kk; t += nt) {
      blo[t] = gl - 4.0 * eps * tnorm - 2.0 * pivmin;
      bhi[t] = gu + 4.0 * eps * tnorm + 2.0 * pivmin;
    }
    __syncthreads();
    if (P == 1) {
      for (int t = tid; t < kk; t += nt) {
        const int idx = n - 1 - t;
        double lo = blo[t], hi = bhi[t];
        for (int it = 0; it < 256; ++it) {
          const double tol = 2.0 * eps * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin;
          if (hi - lo <= tol) break;
          const double mid = 0.5 * (lo + hi);
          if (mid <= lo || mid >= hi) break;
          if (sturm_count_less(dd, e2, n, mid, pivmin) > idx) hi = mid;
          else lo = mid;
        }
        lam[t] = 0.5 * (lo + hi);
      }
    } else {
      const int t = tid / P, g = tid % P;
      const bool mine = t < kk;
      for (int round = 0; round < 256; ++round) {
        bool active = false;
        double x = 0.0;
        if (mine) {
          const double lo = blo[t], hi = bhi[t];
          const double tol = 2.0 * eps * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin;
          x = lo + (hi - lo) * (double)(g + 1) / (double)(P + 1);
          active = hi - lo > tol && x > lo && x < hi;
          cnt[t * P + g] = active ? sturm_count_less(dd, e2, n, x, pivmin) : -1;
        }
        if (!__syncthreads_or(active)) break;
        if (mine && g == 0) {
          const int idx = n - 1 - t;
          const double lo = blo[t], hi = bhi[t];
          // points are increasing; inactive ones (rounded onto an end of
          // the bracket, or a converged bracket) carry no information
          double nlo = lo, nhi = hi;
          for (int q = 0; q < P; ++q) {
            const int c = cnt[t * P + q];
            if (c < 0) continue;
            const double xq = lo + (hi - lo) * (double)(q + 1) / (double)(P + 1);
            if (c > idx) {
              nhi = xq;
              break;
            }
            nlo = xq;
          }
          blo[t] = nlo;
          bhi[t] = nhi;
        }
        __syncthreads();
      }
      for (int tt = tid; tt < kk; tt += nt) lam[tt] = 0.5 * (blo[tt] + bhi[tt]);
    }
  }
  __syncthreads();

  // clusters (dstein: ORTOL = 1e-3 * ||T||_1) and perturbed shifts
  if (tid == 0) {
    double onenrm = 0.0;
    for (int i = 0; i < n; ++i)
      onenrm = fmax(onenrm, fabs(dd[i]) + fabs(ee[i]) + (i > 0 ? fabs(ee[i - 1]) : 0.0));
    const double ortol = 1e-3 * onenrm;
    const double pertol = 10.0 * eps * onenrm;
    int cs = 0;
    for (int t = 0; t < kk; ++t) {
      double s = lam[t];
      if (t > 0) {
        if (lam[t - 1] - lam[t] > ortol) cs = t;
        if (shift[t - 1] - s < pertol) s = shift[t - 1] - pertol;
      }
      shift[t] = s;
      cstart[t] = cs;
    }
  }
  __syncthreads();

  if (J.vals_only) {  // two-stage path: clusters for k_band_mgs / band inverse iteration
    for (int t = tid; t < kk; t += nt) {
      J.shifts[t] = shift[t];
      J.cstarts[t] = cstart[t];
    }
  }
  if (J.vals_only == 1) {  // vectors come from the band matrix
    for (int t = tid; t < kk; t += nt) {
      J.lam[t] = lam[t];
      J.shifts[t] = shift[t];
      J.cstarts[t] = cstart[t];
    }
    return;
  }
  const double tiny = eps * tnorm;
  // start vectors (deterministic pseudo-random, dstein uses dlarnv uniform(-1,1))
  for (int t = tid; t < kk; t += nt) {
    double* z = J.Z + (long long)t * J.ldz;
    for (int r = 0; r < n; ++r) {
      const unsigned h = hash32((unsigned)r * 2654435761u ^ hash32((unsigned)t + 0x9e3779b9u));
      z[r] = ((double)h / 4294967296.0) * 2.0 - 1.0;
    }
  }
  __syncthreads();

  for (int it = 0; it < 3; ++it) {
    for (int t = tid; t < kk; t += nt) {
      const double s = shift[t];
      double* z = J.Z + (long long)t * J.ldz;
      double* Dw = J.piv + (long long)t * n;
      double D = guard_pivot(dd[0] - s, tiny);
      Dw[0] = D;
      double y = z[0];
      for (int r = 1; r < n; ++r) {
        const double l = ee[r - 1] / D;
        D = guard_pivot(dd[r] - s - l * ee[r - 1], tiny);
        Dw[r] = D;
        y = z[r] - l * y;
        z[r] = y;
      }
      double zr = z[n - 1] / Dw[n - 1];
      z[n - 1] = zr;
      double nrm2 = zr * zr;
      for (int r = n - 2; r >= 0; --r) {
        zr = (z[r] - ee[r] * zr) / Dw[r];
        z[r] = zr;
        nrm2 += zr * zr;
      }
      double sc = 1.0 / sqrt(nrm2);
      if (!isfinite(sc) || nrm2 == 0.0) sc = 0.0;
      for (int r = 0; r < n; ++r) z[r] *= sc;
      if (sc == 0.0) z[t % n] = 1.0;
    }
    __syncthreads();
    if (it == 0 || J.vals_only == 2) continue;
    // Gram-Schmidt (twice) inside clusters, in eigenvalue order
    for (int t = 0; t < kk; ++t) {
      const int cs = cstart[t];
      if (cs == t) continue;
      double* zt = J.Z + (long long)t * J.ldz;
      for (int rep = 0; rep < 2; ++rep) {
        for (int c = cs + warp; c < t; c += nwarps) {
          const double* zc = J.Z + (long long)c * J.ldz;
          double s = 0.0;
          for (int r = lane; r < n; r += 32) s += zc[r] * zt[r];
          s = warp_sum(s);
          if (lane == 0) dots[c - cs] = s;
        }
        __syncthreads();
        for (int r = tid; r < n; r += nt) {
          double a = zt[r];
          for (int c = cs; c < t; ++c) a -= dots[c - cs] * J.Z[r + (long long)c * J.ldz];
          zt[r] = a;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int r = tid; r < n; r += nt) part += zt[r] * zt[r];
      const double nrm2 = block_sum(part, red);
      const double sc = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
      for (int r = tid; r < n; r += nt) zt[r] *= sc;
      __syncthreads();
    }
  }
  for (int t = tid; t < kk; t += nt) J.lam[t] = lam[t];
}

// ---------------------------------------------------------------------------
// 3. compact-WY preparation: V in place in A, T per block of NB reflectors
// ---------------------------------------------------------------------------

// (V is made explicit in place by k_prep_v_off: column j of A, rows
// j+off.., becomes reflector v_j.)

// T factor (dlarft, forward, columnwise) of every reflector block of NBT
// reflectors, from S = V^T V (computed by a grouped DMMA GEMM beforehand).
constexpr int NBT = 128;

__global__ void __launch_bounds__(NBT) k_build_t(const EigDev* __restrict__ jobs, int off) {
  const EigDev J = jobs[blockIdx.y];
  const int b = blockIdx.x;
  const int nref = J.n - off;
  const int j0 = b * NBT;
  if (j0 >= nref) return;
  const int nb = min(NBT, nref - j0);
  extern __shared__ double sm[];
  double* T = sm;                      // NBT x (NBT+1), row i at T[i*(NBT+1)]
  double* tau = T + NBT * (NBT + 1);
  const double* S = J.S + (long long)b * NBT * NBT;  // column-major, ld NBT
  const int tid = threadIdx.x;
  tau[tid] = tid < nb ? J.tau[j0 + tid] : 0.0;
  for (int e = tid; e < NBT * (NBT + 1); e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  for (int t = 0; t < nb; ++t) {
    // T[i,t] = -tau_t * sum_{l=i}^{t-1} T[i,l] S[l,t]
    if (tid < t) {
      double s = 0.0;
      for (int l = tid; l < t; ++l) s += T[tid * (NBT + 1) + l] * S[l + t * NBT];
      T[tid * (NBT + 1) + t] = -tau[t] * s;
    }
    if (tid == 0) T[t * (NBT + 1) + t] = tau[t];
    __syncthreads();
  }
  double* out = J.T + (long long)b * NBT * NBT;
  for (int e = tid; e < NBT * NBT; e += blockDim.x) {
    const int i = e % NBT, j = e / NBT;  // column-major
    out[e] = T[i * (NBT + 1) + j];
  }
}

// ---------------------------------------------------------------------------
// Two-stage reduction (large n): dense -> band B2 by panel QR + DMMA GEMMs,
// band -> tridiagonal by Householder bulge chasing (eigenvalues only),
// eigenvectors by inverse iteration on the band matrix, back-transform
// through the stage-1 reflectors (tools/proto/two_stage.py is the numpy
// model of every step; the pipelined chase order was checked there to give
// the sequential result bit for bit).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double& band_at(double* bb, int i, int j) {
  return bb[(i - j) + (long long)j * LDBB];
}

// Panel j0: copy the diagonal block to the band, Householder QR of the
// panel below the band (R -> band, explicit V in place and in VW/WV), T.
__global__ void __launch_bounds__(512, 1) k_panel_qr(const EigDev* __restrict__ jobs, int j0,
                                                     int CS, int vcol) {
  // One matrix per cluster of CS CTAs; CTA c keeps rows [c*mc, (c+1)*mc) of
  // the m x B2 panel in shared memory (column-major, ld mc + 1) for the whole
  // factorisation.  Per column: the norm and the B2-1 column dots are summed
  // from per-CTA partials exchanged through distributed shared memory (every
  // CTA writes its partials into every peer, one cluster barrier, then each
  // sums them in rank order -- identical values in every CTA).
  const EigDev J = jobs[blockIdx.x / CS];
  const int crank = blockIdx.x % CS;
  cg::cluster_group cluster = cg::this_cluster();
  const int n = J.n;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  double* A = J.A;
  const long long lda = J.lda;
  const int jb = max(0, min(B2, n - j0));
  const int r0 = j0 + B2;
  const int m = max(0, n - r0);
  const int mc = (m + CS - 1) / CS;          // rows per CTA
  const int lo = min(m, crank * mc), hi = min(m, lo + mc), ml = hi - lo;
  const int ldp = mc + 1;
  extern __shared__ double psm[];
  double* Pl = psm;                          // [B2][ldp]
  double* xbuf = Pl + (size_t)B2 * ldp;      // [CS][2]   norm partial, alpha
  double* dbuf = xbuf + 2 * CS;              // [CS][B2]  column-dot partials
  __shared__ double beta_s[B2], tau_s[B2], red[32];
  __shared__ double S[B2][B2 + 1], T[B2][B2 + 1];
  cluster.sync();  // peers' shared memory is live before any DSMEM write
  if (j0 >= n) {
    cluster.sync();
    return;
  }
  if (crank == 0)
    for (int e = tid; e < jb * jb; e += nt) {
      const int t = e / jb, i = e % jb;
      if (i >= t) band_at(J.band, j0 + i, j0 + t) = A[(j0 + i) + (long long)(j0 + t) * lda];
    }
  const int nr = m >= 2 ? min(jb, m - 1) : 0;
  double* P = A + r0 + (long long)j0 * lda;
  // panel rows -> shared memory
  for (int e = tid; e < jb * ml; e += nt) {
    const int t = e / ml, i = e % ml;
    Pl[t * ldp + i] = P[lo + i + (long long)t * lda];
  }
  __syncthreads();
  for (int t = 0; t < nr; ++t) {
    double* pt = Pl + t * ldp;
    // (a) norm of rows t+1.. and alpha = P[t][t]
    double part = 0.0;
    for (int i = max(0, t + 1 - lo) + tid; i < ml; i += nt) part += pt[i] * pt[i];
    part = block_sum(part, red);
    const bool own_t = t >= lo && t < hi;
    if (tid == 0)
      for (int c = 0; c < CS; ++c) {
        double* px = cluster.map_shared_rank(xbuf, c);
        px[2 * crank] = part;
        if (own_t) px[1] = pt[t - lo];  // slot 1 of rank 0's pair is unused
      }
    cluster.sync();
    double xn2 = 0.0;
    for (int c = 0; c < CS; ++c) xn2 += xbuf[2 * c];
    const double alpha = xbuf[1];
    double tau = 0.0, beta = alpha, scal = 0.0;
    if (xn2 > 0.0) {
      const double nrm = sqrt(alpha * alpha + xn2);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = max(0, t + 1 - lo) + tid; i < ml; i += nt) pt[i] *= scal;
    if (tid == 0) {
      beta_s[t] = beta;
      tau_s[t] = tau;
      if (crank == 0) J.tau[j0 + t] = tau;
    }
    __syncthreads();
    // (c) s_u = P[t][u] + sum_{i>t} v_i P[i][u] for u > t (partials)
    for (int u = t + 1 + warp; u < jb; u += nwarps) {
      const double* pu = Pl + u * ldp;
      double sp = 0.0;
      for (int i = max(0, t + 1 - lo) + lane; i < ml; i += 32) sp += pt[i] * pu[i];
      sp = warp_sum(sp);
      if (own_t) sp += pu[t - lo];
      if (lane < CS) cluster.map_shared_rank(dbuf, lane)[crank * B2 + u] = sp;
    }
    cluster.sync();
    // (d) P[i][u] -= tau s_u v_i
    if (tau != 0.0) {
      for (int u = t + 1 + warp; u < jb; u += nwarps) {
        double su = 0.0;
        for (int c = 0; c < CS; ++c) su += dbuf[c * B2 + u];
        su *= tau;
        double* pu = Pl + u * ldp;
        if (own_t && lane == 0) pu[t - lo] -= su;
        for (int i = max(0, t + 1 - lo) + lane; i < ml; i += 32) pu[i] -= su * pt[i];
      }
    }
    __syncthreads();
  }
  if (tid < B2 && tid >= nr) {
    tau_s[tid] = 0.0;
    if (crank == 0 && tid < jb) J.tau[j0 + tid] = 0.0;
  }
  __syncthreads();
  // R -> band (panel rows i <= t < B2, owned by the CTAs holding rows < B2)
  for (int e = tid; e < jb * jb; e += nt) {
    const int t = e / jb, i = e % jb;
    if (i <= t && i < m && i >= lo && i < hi)
      band_at(J.band, r0 + i, j0 + t) = (i == t && t < nr) ? beta_s[t] : Pl[t * ldp + i - lo];
  }
  // explicit V (unit lower trapezoidal) in place, in the VW / WV panels and
  // in shared memory (for V^T V)
  __syncthreads();
  for (int e = tid; e < jb * ml; e += nt) {
    const int t = e / ml, i = e % ml, ig = lo + i;
    const double v = t >= nr ? 0.0 : (ig < t ? 0.0 : (ig == t ? 1.0 : Pl[t * ldp + i]));
    Pl[t * ldp + i] = v;
    P[ig + (long long)t * lda] = v;
    J.VW[(r0 + ig) + (long long)(vcol + t) * n] = v;
    J.WV[(r0 + ig) + (long long)(vcol + B2 + t) * n] = v;
  }
  __syncthreads();
  // S = V^T V: partials of the local rows into rank 0
  // (partials through global memory: CS x B2^2 doubles would not fit next to
  // the panel at the largest n; rank 0 sums them in rank order after the
  // cluster barrier, reading through L2)
  double* s0 = J.psum + (size_t)crank * B2 * B2;
  for (int pq = warp; pq < B2 * B2; pq += nwarps) {
    const int pp = pq / B2, q = pq % B2;
    if (pp > q) continue;
    double sp = 0.0;
    if (q < nr) {
      const double* vp = Pl + pp * ldp;
      const double* vq = Pl + q * ldp;
      for (int i = max(0, q - lo) + lane; i < ml; i += 32) sp += vp[i] * vq[i];
      sp = warp_sum(sp);
    }
    if (lane == 0) s0[pq] = sp;
  }
  cluster.sync();  // last DSMEM access: peers may exit after this
  if (crank != 0) return;
  for (int pq = tid; pq < B2 * B2; pq += nt) {
    const int pp = pq / B2, q = pq % B2;
    double sv = 0.0;
    if (pp <= q)
      for (int c = 0; c < CS; ++c) sv += __ldcg(J.psum + (size_t)c * B2 * B2 + pq);
    S[pp][q] = sv;
  }
  for (int e = tid; e < B2 * (B2 + 1); e += nt) (&T[0][0])[e] = 0.0;
  __syncthreads();
  for (int t = 0; t < B2; ++t) {
    if (tid < t) {
      double sv = 0.0;
      for (int l = tid; l < t; ++l) sv += T[tid][l] * S[l][t];
      T[tid][t] = -tau_s[t] * sv;
    }
    if (tid == 0) T[t][t] = tau_s[t];
    __syncthreads();
  }
  double* out = J.Tp + (long long)(j0 / B2) * B2 * B2;
  for (int e = tid; e < B2 * B2; e += nt) out[e] = T[e % B2][e / B2];
}

constexpr size_t kPanelSmemMax = 200 * 1024;
size_t panel_smem(int mc, int cs) {
  return ((size_t)B2 * (mc + 1) + 2 * cs + (size_t)cs * B2) * sizeof(double);
}

void launch_panel_qr(Ctx& ctx, int count, int mmax, const EigDev* dd, int j0, int vcol) {
  int cs = 1;
  while (cs < 8 && panel_smem((mmax + cs - 1) / cs, cs) > kPanelSmemMax) cs *= 2;
  const size_t smem = panel_smem((mmax + cs - 1) / cs, cs);
  if (smem > kPanelSmemMax) throw Error(kInvalid, "k_panel_qr: n too large");
  smem_optin(k_panel_qr, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ctx.launch_begin();
  HSVD_CUDA(cudaLaunchKernelEx(&cfg, k_panel_qr, dd, j0, cs, vcol));
  ctx.check_launch("k_panel_qr");
}

// WV[:, vcol:vcol+B2] = W (= VW[:, vcol+B2:vcol+2B2]) for the rows below the panel
// (panels with no trailing matrix, r0 > n-2: W := 0 on the rows r0..n-1, so
// the pending pairs of the group stay finite and exact)
__global__ void k_copy_w(const EigDev* __restrict__ jobs, int j0, int vcol) {
  const EigDev J = jobs[blockIdx.y];
  const int n = J.n, r0 = j0 + B2;
  if (r0 > n - 2) {
    if (blockIdx.x == 0)
      for (int e = threadIdx.x; e < max(0, n - r0) * B2; e += blockDim.x) {
        const int i = r0 + e % max(1, n - r0), t = e / max(1, n - r0);
        J.WV[i + (long long)(vcol + t) * n] = 0.0;
        J.VW[i + (long long)(vcol + B2 + t) * n] = 0.0;
      }
    return;
  }
  const long long total = (long long)(n - r0) * B2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = r0 + (int)(e % (n - r0)), t = (int)(e / (n - r0));
    J.WV[i + (long long)(vcol + t) * n] = J.VW[i + (long long)(vcol + B2 + t) * n];
  }
}

// Band -> tridiagonal by Householder bulge chasing (eigenvalues only).
// One CTA per matrix; warp w runs sweeps w, w+W, ...; sweep s may do step
// k only after sweep s-1 finished step k+3 (or the whole sweep), which
// reproduces the sequential result exactly.
__device__ __forceinline__ unsigned long long prog_encode(int s, unsigned steps) {
  return ((unsigned long long)(unsigned)(s + 1) << 32) | steps;
}
constexpr unsigned kSweepDone = 0x7fffffffu;

constexpr int CHASE_WARPS = 8;
static_assert(B2 == 32, "k_chase maps one band row per lane");

// One bulge-chasing step of a warp: reflector from column c (rows r0..r0+L),
// applied to the left block (columns c+1..c+nl), two-sided to the L x L
// block R at r0 and from the right to the na rows below R.  Every element
// is addressed from a per-lane base pointer plus a compile-time offset
// (band column stride LDBB, diagonal stride LDBB-1); FULL (L == B2 and
// nl == B2-1) drops the per-column bounds.  Returns false when the column
// is already reduced (the sweep ends).
template <bool CG>
__device__ __forceinline__ double band_ld(const double* p) {
  return CG ? __ldcg(p) : *p;
}

// Steps of sweep s (k with r0 = s+1+32k <= n-2) and the steps of all sweeps
// before it: the compact sweep-major index of the stored chase reflectors.
__device__ __forceinline__ int sweep_steps(int n, int s) { return (n - 3 - s) / B2 + 1; }
__device__ __forceinline__ long long floor_sum(long long A) {  // sum_{a=0}^{A} floor(a/B2)
  if (A < 0) return 0;
  const long long q = (A + 1) / B2, r = (A + 1) % B2;
  return B2 * q * (q - 1) / 2 + r * q;
}
__device__ __forceinline__ long long steps_before(int n, int s) {
  return s + floor_sum(n - 3) - floor_sum(n - 3 - s);
}

// carry: x and the left block of this step are the rows-after block the
// same warp updated in its previous step (its column 0 and columns 1..31),
// still in registers (x, yl); last: no further step in this sweep, so the
// updated rows-after block is stored instead of being carried.
template <bool FULL, bool CG>
__device__ __forceinline__ bool chase_step(double* bb, int c, int r0, int L, int nl, int na,
                                           int lane, double* vs, double* ws, double* rout,
                                           bool carry, bool last, double& x,
                                           double (&yl)[B2 - 1]) {
  constexpr long long LD = LDBB;
  const bool lx = lane < L;
  double* px = bb + (r0 + lane - c) + (long long)c * LD;
  double* pyl = bb + (r0 + lane - c - 1) + (long long)(c + 1) * LD;
  double* pa1 = bb + lane + (long long)r0 * LD;                 // (r0+lane, r0+j), j <= lane
  double* pa2 = bb + (long long)(r0 + lane) * LD - lane;        // (r0+j, r0+lane), j > lane
  double* pya = bb + (L + lane) + (long long)r0 * LD;           // (r0+L+lane, r0+j)
  const bool ly = lane < na;
  // all loads of the step issued together (one memory round trip); a
  // carried bulge needs none for x and the left block
  double ar[B2], ya[B2];
  if (!carry) {
    x = lx ? band_ld<CG>(px) : 0.0;
#pragma unroll
    for (int l = 0; l < B2 - 1; ++l)
      yl[l] = (lx && (FULL || l < nl)) ? band_ld<CG>(pyl + l * (LD - 1)) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < B2; ++j) {
    const double* pa = lane >= j ? pa1 + j * (LD - 1) : pa2 + j;
    ar[j] = (lx && (FULL || j < L)) ? band_ld<CG>(pa) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < B2; ++j) ya[j] = (ly && (FULL || j < L)) ? band_ld<CG>(pya + j * (LD - 1)) : 0.0;
  const double xn2 = warp_sum(lane >= 1 ? x * x : 0.0);
  const double alpha = __shfl_sync(0xffffffffu, x, 0);
  if (xn2 == 0.0) {  // no bulge left: a carried block still has to reach memory
    if (carry) {
      if (lx) *px = x;
#pragma unroll
      for (int l = 0; l < B2 - 1; ++l)
        if (lx && (FULL || l < nl)) pyl[l * (LD - 1)] = yl[l];
    }
    return false;
  }
  const double nrm = sqrt(alpha * alpha + xn2);
  const double beta = alpha >= 0.0 ? -nrm : nrm;
  const double tau = (beta - alpha) / beta;
  const double scal = 1.0 / (alpha - beta);
  const double v = lane == 0 ? 1.0 : (lx ? x * scal : 0.0);
  vs[lane] = v;
  if (rout) {  // kept for the eigenvector back-transform (k_q2_apply)
    __stcs(rout + lane, v);  // streaming: read once by k_q2_apply, keep L2 for the band
    if (lane == 0) __stcs(rout + B2, tau);
  }
  if (lx) *px = lane == 0 ? beta : 0.0;
  // left block: d_l = sum_i v_i y_il by a transposing butterfly (lane l
  // ends with d_l), then y_il -= tau v_i d_l
  {
    double t[B2];
#pragma unroll
    for (int l = 0; l < B2 - 1; ++l) t[l] = v * yl[l];
    t[B2 - 1] = 0.0;
#pragma unroll
    for (int ofs = 16; ofs >= 1; ofs >>= 1) {
      const bool up = (lane & ofs) != 0;
#pragma unroll
      for (int j = 0; j < ofs; ++j) {
        const double send = up ? t[j] : t[j + ofs];
        const double got = __shfl_xor_sync(0xffffffffu, send, ofs);
        t[j] = (up ? t[j + ofs] : t[j]) + got;
      }
    }
    const double dl = tau * t[0];
#pragma unroll
    for (int l = 0; l < B2 - 1; ++l) {
      const double d = __shfl_sync(0xffffffffu, dl, l);
      if (lx && (FULL || l < nl)) pyl[l * (LD - 1)] = yl[l] - d * v;
    }
  }
  __syncwarp();
  // R x R: two-sided (symmetric, lower storage); p = tau R v
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
  for (int j = 0; j < B2; j += 4) {
    p0 += ar[j] * vs[j];
    p1 += ar[j + 1] * vs[j + 1];
    p2 += ar[j + 2] * vs[j + 2];
    p3 += ar[j + 3] * vs[j + 3];
  }
  const double pp = tau * ((p0 + p1) + (p2 + p3));
  const double al = -0.5 * tau * warp_sum(pp * v);
  const double w = pp + al * v;
  ws[lane] = w;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < B2; ++j)
    if (lx && lane >= j && (FULL || j < L)) pa1[j * (LD - 1)] = ar[j] - (v * ws[j] + w * vs[j]);
  // rows after R: right application (creates the next bulge)
  double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
  for (int j = 0; j < B2; j += 4) {
    y0 += ya[j] * vs[j];
    y1 += ya[j + 1] * vs[j + 1];
    y2 += ya[j + 2] * vs[j + 2];
    y3 += ya[j + 3] * vs[j + 3];
  }
  const double y = tau * ((y0 + y1) + (y2 + y3));
  if (last) {
#pragma unroll
    for (int j = 0; j < B2; ++j)
      if (ly && (FULL || j < L)) pya[j * (LD - 1)] = ya[j] - y * vs[j];
  } else {  // the next step's x and left block (stored by that step)
    x = ya[0] - y * vs[0];
#pragma unroll
    for (int l = 0; l < B2 - 1; ++l) yl[l] = (FULL || l + 1 < L) ? ya[l + 1] - y * vs[l + 1] : 0.0;
  }
  return true;
}

// The sweeps of one matrix run on a cluster of CS CTAs (CS * CHASE_WARPS
// warps; sweep s on global warp s mod (CS * CHASE_WARPS)).  Progress flags
// live in each CTA's shared memory and are polled through DSMEM; with CS > 1
// the band is read through L2 (__ldcg), since a peer SM may have rewritten a
// line this SM's L1 still holds, and every step's stores are fenced at gpu
// scope before its flag is published.
template <bool CL>
__global__ void __launch_bounds__(CHASE_WARPS * 32, 1) k_chase(const EigDev* __restrict__ jobs,
                                                              int CS) {
  const int crank = CL ? (int)(blockIdx.x % CS) : 0;
  const EigDev J = jobs[CL ? blockIdx.x / CS : blockIdx.x];
  const int n = J.n;
  double* bb = J.band;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = CHASE_WARPS * (CL ? CS : 1);   // warps working on this matrix
  const int gw = crank * CHASE_WARPS + warp;    // this warp's global index
  __shared__ unsigned long long prog[CHASE_WARPS];
  __shared__ double vsh[CHASE_WARPS][B2];
  __shared__ double wsh[CHASE_WARPS][B2];
  if (tid < CHASE_WARPS) prog[tid] = prog_encode(crank * CHASE_WARPS + tid - W, kSweepDone);
  cg::cluster_group cluster = cg::this_cluster();
  if (CL) cluster.sync();
  else __syncthreads();
  const int pg = (gw - 1 + W) % W;  // warp running sweep s-1
  volatile unsigned long long* pprog =
      CL ? cluster.map_shared_rank(prog, pg / CHASE_WARPS) + pg % CHASE_WARPS : prog + pg;
  volatile unsigned long long* myprog = prog + warp;
  // release-store of this warp's progress (cluster scope: the consumer may
  // run on the peer SM and reads the band through L2 after its acquire)
  auto publish = [&](unsigned long long val) {
    if (CL) {
      if (lane == 0)
        asm volatile("st.release.cluster.u64 [%0], %1;\n" ::"l"(myprog), "l"(val) : "memory");
    } else {
      __threadfence_block();
      if (lane == 0) *myprog = val;
    }
  };
  unsigned long long seen = 0;  // last acquired progress of sweep s-1's warp
  const int nsweeps = n - 2;
  for (int s = gw; s < nsweeps; s += W) {
    double cx, cyl[B2 - 1];  // x and left block, carried between consecutive steps
    for (int k = 0;; ++k) {
      const int r0 = s + 1 + k * B2;
      if (r0 >= n) break;
      const int r1 = min(n, r0 + B2), L = r1 - r0;
      if (L < 2) break;
      if (s > 0) {  // wait for sweep s-1 to be 3 steps ahead (or done)
        const unsigned need = (unsigned)(k + 3);
        auto ahead = [&](unsigned long long pv) {
          const int vs = (int)(pv >> 32) - 1;
          const unsigned st = (unsigned)(pv & 0xffffffffu);
          return vs > s - 1 || (vs == s - 1 && st >= need);
        };
        // progress only grows: a value already acquired that suffices needs
        // no new (remote) poll
        if (!ahead(seen)) {
          while (true) {
            unsigned long long pv;
            if (CL)
              asm volatile("ld.acquire.cluster.u64 %0, [%1];\n"
                           : "=l"(pv)
                           : "l"(pprog)
                           : "memory");
            else
              pv = *pprog;
            if (ahead(pv)) {
              seen = pv;
              break;
            }
            __nanosleep(100);
          }
          if (!CL) __threadfence_block();
        }
      }
      const int c = k == 0 ? s : s + 1 + (k - 1) * B2;
      const int nl = r0 - c - 1;                // left-block columns (0 or B2-1)
      const int na = min(n, r0 + 2 * B2) - r1;  // rows after R
      double* rout = J.refl ? J.refl + (steps_before(n, s) + k) * (B2 + 1) : nullptr;
      const bool last = r0 + B2 > n - 2;  // the loop's own continuation test
      const bool ok =
          (L == B2 && nl == B2 - 1)
              ? chase_step<true, CL>(bb, c, r0, L, nl, na, lane, vsh[warp], wsh[warp], rout,
                                     k > 0, last, cx, cyl)
              : chase_step<false, CL>(bb, c, r0, L, nl, na, lane, vsh[warp], wsh[warp], rout,
                                      k > 0, last, cx, cyl);
      if (!ok) {  // no bulge left in this sweep: its remaining reflectors are I
        if (J.refl && lane == 0)
          for (int k2 = k; k2 < sweep_steps(n, s); ++k2)
            J.refl[(steps_before(n, s) + k2) * (B2 + 1) + B2] = 0.0;
        break;
      }
      __syncwarp();  // every lane's band stores before lane 0's release
      publish(prog_encode(s, (unsigned)(k + 1)));
    }
    __syncwarp();
    publish(prog_encode(s, kSweepDone));
  }
  if (CL) {
    __threadfence();
    cluster.sync();  // every sweep done; no DSMEM access after this
    if (crank != 0) return;
  } else {
    __syncthreads();
  }
  for (int i = tid; i < n; i += blockDim.x) {
    J.d[i] = band_ld<CL>(&band_at(bb, i, i));
    if (i < n - 1) J.e[i] = band_ld<CL>(&band_at(bb, i + 1, i));
  }
}

// Eigenvectors of the band matrix from those of its tridiagonal: Z <- Q2 Z
// with Q2 the product of the chase reflectors in chase order, applied in
// reverse (LAPACK dsbtrd's Q, applied as dormtr would).  Every reflector
// re-reads and rewrites its 32 rows of Z, so the rows must live on chip: one
// CTA per NC eigenvectors keeps its n x NC slice of Z in shared memory for
// the whole pass (row-major; lane = column x row group, rows interleaved so
// a warp's accesses are conflict-free).  The reflectors of one sweep touch
// disjoint 32-row blocks: the CTA's 8 warps share a sweep's blocks and
// synchronise once per sweep, with the next sweep's reflectors staged into
// shared memory by cp.async while the current one is applied.
constexpr int Q2_WARPS = 8;

template <int NC>
__global__ void __launch_bounds__(Q2_WARPS * 32) k_q2_apply(const EigDev* __restrict__ jobs) {
  constexpr int G = 32 / NC;       // row groups per warp
  constexpr int RPL = B2 / G;      // rows per lane
  const EigDev J = jobs[blockIdx.y];
  const int n = J.n, kk = J.kk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  const int c0 = blockIdx.x * NC;
  if (c0 >= kk || n < 3) return;
  const int nc = min(NC, kk - c0);
  const int kmax = sweep_steps(n, 0);
  extern __shared__ __align__(16) double q2sm[];
  double* Zs = q2sm;                              // [n][NC]
  double* rbuf = q2sm + (size_t)n * NC;           // [2][kmax][B2 + 1]
  for (int e = tid; e < n * NC; e += nt) {
    const int r = e % n, q = e / n;
    Zs[r * NC + q] = q < nc ? J.Z[r + (long long)(c0 + q) * J.ldz] : 0.0;
  }
  const double* R = J.refl;
  auto stage = [&](int s, int buf) {
    const double* src = R + steps_before(n, s) * (B2 + 1);
    double* dst = rbuf + (size_t)buf * kmax * (B2 + 1);
    const int cnt = sweep_steps(n, s) * (B2 + 1);
    for (int e = tid; e < cnt; e += nt) {
      const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst + e));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src + e));
    }
  };
  stage(n - 3, 0);
  asm volatile("cp.async.commit_group;\n");
  const int q = lane % NC, g = lane / NC;  // column, row group
  int it = 0;
  for (int s = n - 3; s >= 0; --s, ++it) {
    const int sb = it & 1;
    if (s > 0) stage(s - 1, sb ^ 1);
    asm volatile("cp.async.commit_group;\n");
    asm volatile("cp.async.wait_group 1;\n");
    __syncthreads();
    const double* rb = rbuf + (size_t)sb * kmax * (B2 + 1);
    const int K = sweep_steps(n, s);
    for (int k = warp; k < K; k += Q2_WARPS) {
      const double* rv = rb + k * (B2 + 1);
      const double tau = rv[B2];
      if (tau == 0.0) continue;
      const int r0 = s + 1 + k * B2, L = min(B2, n - r0);
      double z[RPL], v[RPL];
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int i = g + G * j;  // row of the block
        v[j] = rv[i];
        z[j] = i < L ? Zs[(r0 + i) * NC + q] : 0.0;
      }
      double dot = 0.0;
#pragma unroll
      for (int j = 0; j < RPL; ++j) dot += v[j] * z[j];
#pragma unroll
      for (int o = NC; o < 32; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      dot *= tau;
#pragma unroll
      for (int j = 0; j < RPL; ++j) {
        const int i = g + G * j;
        if (i < L) Zs[(r0 + i) * NC + q] = z[j] - dot * v[j];
      }
    }
    __syncthreads();  // next sweep: rows overlap, and this buffer is restaged
  }
  asm volatile("cp.async.wait_group 0;\n");
  __syncthreads();
  for (int e = tid; e < n * NC; e += nt) {
    const int r = e % n, qq = e / n;
    if (qq < nc) J.Z[r + (long long)(c0 + qq) * J.ldz] = Zs[r * NC + qq];
  }
}

// Columns per CTA: as many as fit shared memory with the reflector buffers.
int q2_cols(int n) {
  const size_t rb = (size_t)2 * ((n - 3) / B2 + 1) * (B2 + 1) * sizeof(double);
  for (int nc : {8, 4, 2})
    if ((size_t)n * nc * sizeof(double) + rb <= 220 * 1024) return nc;
  return 0;
}

size_t q2_smem(int n, int nc) {
  return (size_t)n * nc * sizeof(double) + (size_t)2 * ((n - 3) / B2 + 1) * (B2 + 1) * sizeof(double);
}

// Eigenvectors of the band matrix (band0, bandwidth B2) by inverse
// iteration, one warp per shift on a (cpm x count) grid.  The warp factors
// (B - shift I) = P L U with partial pivoting in a (B2+1) x (2*B2+1)
// shared-memory window (entering band rows prefetched two steps ahead),
// streaming U rows and multipliers to its workspace; then three
// forward/backward solves.  The solves keep the live part of the vector in
// a 128-entry shared ring and prefetch U / L rows and vector entries one
// INV_PF-step chunk ahead, so their step chain never waits on HBM.
// k_band_mgs orthogonalises inside eigenvalue clusters afterwards.
__device__ __forceinline__ double band_full(const double* b0, int n, int i, int j) {
  if (i < 0 || j < 0 || i >= n || j >= n) return 0.0;
  const int d = i - j;
  if (d > B2 || d < -B2) return 0.0;
  return d >= 0 ? b0[d + (long long)j * LDBB] : b0[-d + (long long)i * LDBB];
}

constexpr int INV_PF = 8;      // solve prefetch chunk (steps)
constexpr int INV_RING = 128;  // vector ring entries per warp (>= 2*B2+1)

__device__ __forceinline__ double invit_start(int r, int t) {
  const unsigned h = hash32((unsigned)r * 2654435761u ^ hash32((unsigned)t + 0x9e3779b9u));
  return ((double)h / 4294967296.0) * 2.0 - 1.0;
}

__global__ void __launch_bounds__(INV_WARPS * 32, 3) k_band_invit(const EigDev* __restrict__ jobs) {
  const EigDev J = jobs[blockIdx.y];
  const int n = J.n, kk = J.kk;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  constexpr int WR = B2 + 1, WC = 2 * B2 + 1;  // window rows / columns
  extern __shared__ double sm[];
  double* win = sm + (size_t)warp * WR * WC;
  double* yw = sm + (size_t)INV_WARPS * WR * WC + (size_t)warp * INV_RING;
  double* red = sm + (size_t)INV_WARPS * (WR * WC + INV_RING);
  const double* b0 = J.band0;
  // ||B||_inf for the pivot guard
  double nb = 0.0;
  for (int i = tid; i < n; i += nt) {
    double s = 0.0;
    for (int j = max(0, i - B2); j <= min(n - 1, i + B2); ++j) s += fabs(band_full(b0, n, i, j));
    nb = fmax(nb, s);
  }
  const double bnorm = block_max(nb, red);
  const double tiny = DBL_EPSILON * fmax(bnorm, DBL_MIN);
  const int gw = blockIdx.x * INV_WARPS + warp, nw_total = gridDim.x * INV_WARPS;
  // workspace of this warp: U rows (n x WC), multipliers (n x B2), pivots,
  // forward result F, iterate X
  double* U = J.lu + ((size_t)blockIdx.y * nw_total + gw) * (size_t)J.lu_slot;
  double* Lm = U + (size_t)n * WC;
  int* piv = reinterpret_cast<int*>(Lm + (size_t)n * B2);
  double* F = Lm + (size_t)n * B2 + n;
  double* X = F + n;
  for (int t = gw; t < kk; t += nw_total) {
    const double sh = J.shifts[t];
    // ---- factorisation: window rows are slots (row % WR), columns (col % WC)
    for (int e = lane; e < WR * WC; e += 32) win[e] = 0.0;
    __syncwarp();
    for (int i = 0; i <= B2 && i < n; ++i)
      for (int c = lane; c <= 2 * B2; c += 32)
        if (c < n) win[(i % WR) * WC + (c % WC)] = band_full(b0, n, i, c) - (i == c ? sh : 0.0);
    __syncwarp();
    double preA[3], preB[3];
    // band row rn = jj + B2 + 1 at columns jj+1+cc, cc = lane + 32q: q = 0
    // the strictly lower part (diagonal B2-lane of column rn-B2+lane), q = 1
    // diagonal and upper part (column rn of the band, mirrored), q = 2
    // (lane 0) the last upper element
    auto fetch_row = [&](double* pre, int rn) {
      const bool in = rn < n;
      const double* crn = b0 + (long long)rn * LDBB;
      pre[0] = in ? b0[(B2 - lane) + (long long)(rn - B2 + lane) * LDBB] : 0.0;
      pre[1] = (in && rn + lane < n) ? crn[lane] - (lane == 0 ? sh : 0.0) : 0.0;
      pre[2] = (in && lane == 0 && rn + B2 < n) ? crn[B2] : 0.0;
    };
    fetch_row(preA, B2 + 1);
    fetch_row(preB, B2 + 2);
    for (int j = 0; j < n; ++j) {
      const int nw = min(WR, n - j);  // candidate rows j..j+nw-1
      const int cj = j % WC;
      // lane i holds candidate row j+i; lane 0 also row j+B2
      double a = lane < nw ? fabs(win[((j + lane) % WR) * WC + cj]) : -1.0;
      int p = lane;
      if (lane == 0 && nw == WR) {
        const double a2 = fabs(win[((j + B2) % WR) * WC + cj]);
        if (a2 > a) {
          a = a2;
          p = B2;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ao = __shfl_xor_sync(0xffffffffu, a, o);
        const int po = __shfl_xor_sync(0xffffffffu, p, o);
        if (ao > a || (ao == a && po < p)) {
          a = ao;
          p = po;
        }
      }
      const int sj = (j % WR) * WC, sp = ((j + p) % WR) * WC;
      if (p != 0)
        for (int c = lane; c < WC; c += 32) {
          const double tmp = win[sj + c];
          win[sj + c] = win[sp + c];
          win[sp + c] = tmp;
        }
      __syncwarp();
      double u = win[sj + cj];
      if (fabs(u) < tiny) u = u < 0.0 ? -tiny : tiny;
      const double ru = 1.0 / u;
      const int ncol = min(2 * B2, n - 1 - j);
      // columns j+1..j+ncol sit in slots cj+1..WC-1 then 0..(cj+ncol-WC)
      // lane i (1..nw-1) eliminates row j+i over all 2*B2 window columns
      // after j (columns past n hold zeros in both rows), eight at a time
      // with the loads batched ahead of the stores
      if (lane >= 1 && lane < nw) {
        const int si = ((j + lane) % WR) * WC;
        const double l = win[si + cj] * ru;
        double* ri = win + si;
        const double* rp = win + sj;
#pragma unroll
        for (int c0 = 1; c0 <= 2 * B2; c0 += 8) {
          int cc[8];
          double x[8], y[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int c = cj + c0 + q;
            cc[q] = c >= WC ? c - WC : c;
            x[q] = ri[cc[q]];
            y[q] = rp[cc[q]];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) ri[cc[q]] = x[q] - l * y[q];
        }
        Lm[(size_t)j * B2 + (lane - 1)] = l;
      }
      if (nw == WR) {  // row j+B2: its columns split over the lanes
        const int si = ((j + B2) % WR) * WC;
        const double l = win[si + cj] * ru;
        for (int cc = 1 + lane; cc <= ncol; cc += 32) {
          int c = cj + cc;
          c -= c >= WC ? WC : 0;
          win[si + c] -= l * win[sj + c];
        }
        if (lane == 0) Lm[(size_t)j * B2 + (B2 - 1)] = l;
      }
      __syncwarp();
      // column j leaves; its slot becomes column j+2B2+1
      if (lane >= 1 && lane < nw) win[((j + lane) % WR) * WC + cj] = 0.0;
      if (lane == 0 && nw == WR) win[((j + B2) % WR) * WC + cj] = 0.0;
      if (lane == 0) {
        piv[j] = p;
        win[sj + cj] = u;
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int cc = lane + 32 * q;
        if (cc < WC) {
          int c = cj + cc;
          c -= c >= WC ? WC : 0;
          U[(size_t)j * WC + cc] = (cc <= ncol) ? win[sj + c] : 0.0;
        }
      }
      __syncwarp();
      // the slot of row j now holds row j+B2+1 (columns j+1..j+2B2+1)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int cc = lane + 32 * q;
        if (cc < WC) {
          int c = cj + 1 + cc;
          c -= c >= WC ? WC : 0;
          win[sj + c] = preA[q];
        }
      }
#pragma unroll
      for (int q = 0; q < 3; ++q) preA[q] = preB[q];
      fetch_row(preB, j + B2 + 3);
      __syncwarp();
    }
    __syncwarp();
    // ---- three solves; iterate it reads X scaled by sc (it = 0: start vector)
    double sc = 1.0;
    bool unit = false;  // previous iterate degenerate: restart from e_t
    for (int it = 0; it < 3; ++it) {
      auto input = [&](int r) -> double {
        if (r >= n) return 0.0;
        if (it == 0) return invit_start(r, t);
        if (unit) return r == t % n ? 1.0 : 0.0;
        return X[r] * sc;
      };
      // forward: y <- L^-1 P y.  Ring holds y[j..j+B2] before step j.
      for (int r = lane; r <= B2; r += 32) yw[r] = input(r);
      __syncwarp();
      {
        // chunk j0..j0+INV_PF-1: lane d holds the pivot and the entering
        // entry of step j0+d, every lane its multiplier of each step
        double Lc[INV_PF], Ln[INV_PF];
        int pc, pn;
        double ec, en;
        auto load = [&](int j0, double* Lx, int& px, double& ex) {
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) {
            const int j = j0 + d;
            Lx[d] = j < n ? Lm[(size_t)j * B2 + lane] : 0.0;
          }
          const int jl = j0 + lane;
          px = (lane < INV_PF && jl < n) ? piv[jl] : 0;
          ex = lane < INV_PF ? input(jl + B2 + 1) : 0.0;
        };
        load(0, Lc, pc, ec);
        for (int j0 = 0; j0 < n; j0 += INV_PF) {
          load(j0 + INV_PF, Ln, pn, en);
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) {
            const int j = j0 + d;
            const int p = __shfl_sync(0xffffffffu, pc, d);
            const double e = __shfl_sync(0xffffffffu, ec, d);
            if (j < n) {
              if (p != 0 && lane == 0) {
                const double tmp = yw[j & (INV_RING - 1)];
                yw[j & (INV_RING - 1)] = yw[(j + p) & (INV_RING - 1)];
                yw[(j + p) & (INV_RING - 1)] = tmp;
              }
              __syncwarp();
              const double yj = yw[j & (INV_RING - 1)];
              if (j + 1 + lane < n) yw[(j + 1 + lane) & (INV_RING - 1)] -= Lc[d] * yj;
              if (lane == 0) {
                F[j] = yj;
                yw[(j + B2 + 1) & (INV_RING - 1)] = e;
              }
              __syncwarp();
            }
          }
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) Lc[d] = Ln[d];
          pc = pn;
          ec = en;
        }
      }
      __syncwarp();
      // backward: U x = F.  Ring holds x[j+1..j+2B2] before step j.
      for (int r = lane; r < INV_RING; r += 32) yw[r] = 0.0;
      __syncwarp();
      double nrm2 = 0.0;
      {
        // chunk j0, j0-1, ..: lane d holds 1/U[j0-d][0] and F[j0-d]
        double Ac[INV_PF], Bc[INV_PF], An[INV_PF], Bn[INV_PF];
        double rc, fc, rn, fn;
        auto load = [&](int j0, double* Ax, double* Bx, double& rx, double& fx) {
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) {
            const int j = j0 - d;
            const double* ur = U + (size_t)(j >= 0 ? j : 0) * WC;
            Ax[d] = j >= 0 ? ur[1 + lane] : 0.0;
            Bx[d] = j >= 0 ? ur[33 + lane] : 0.0;  // lanes 0..31 -> cc 33..64
          }
          const int jl = j0 - lane;
          const bool ok = lane < INV_PF && jl >= 0;
          rx = ok ? 1.0 / U[(size_t)jl * WC] : 0.0;
          fx = ok ? F[jl] : 0.0;
        };
        load(n - 1, Ac, Bc, rc, fc);
        for (int j0 = n - 1; j0 >= 0; j0 -= INV_PF) {
          load(j0 - INV_PF, An, Bn, rn, fn);
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) {
            const int j = j0 - d;
            const double rj = __shfl_sync(0xffffffffu, rc, d);
            const double fj = __shfl_sync(0xffffffffu, fc, d);
            if (j >= 0) {
              double s = Ac[d] * yw[(j + 1 + lane) & (INV_RING - 1)] +
                         Bc[d] * yw[(j + 33 + lane) & (INV_RING - 1)];
              s = warp_sum(s);
              const double x = (fj - s) * rj;
              // (ring slots of x[j+2B2+1..] are only reused for indices
              // that are written before they are read)
              if (lane == 0) {
                yw[j & (INV_RING - 1)] = x;
                X[j] = x;
              }
              nrm2 += x * x;
              __syncwarp();
            }
          }
#pragma unroll
          for (int d = 0; d < INV_PF; ++d) {
            Ac[d] = An[d];
            Bc[d] = Bn[d];
          }
          rc = rn;
          fc = fn;
        }
      }
      __syncwarp();
      unit = !(nrm2 > 0.0 && isfinite(nrm2));
      sc = unit ? 0.0 : 1.0 / sqrt(nrm2);
    }
    double* z = J.Z + (long long)t * J.ldz;
    for (int r = lane; r < n; r += 32) z[r] = unit ? (r == t % n ? 1.0 : 0.0) : X[r] * sc;
    __syncwarp();
  }
}

// Orthonormalisation of the inverse-iteration vectors inside eigenvalue
// clusters, in eigenvalue order (the result of dstein's modified
// Gram-Schmidt, reorganised for bandwidth): each cluster is processed in
// panels of GS_P vectors; a panel is first projected against all earlier
// vectors of its cluster twice (block classical Gram-Schmidt, 32x32 tiles
// of Z_prev^T Z_panel accumulated through shared memory, so every earlier
// vector is read once per panel rather than once per vector), then its own
// vectors are orthonormalised one by one (classical Gram-Schmidt twice).
// 256 threads; smem: 2*64*33 + 32*33 + 64 doubles.
constexpr int GS_P = 32;
constexpr int GS_R = 64;  // rows per staged tile
constexpr int GS_SMEM_DOUBLES = 2 * GS_R * 33 + GS_P * 33 + 64;

__device__ void cluster_gs(double* Z, long long ldz, int n, int cs, int ce, double* sm) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = nt >> 5;
  double* At = sm;               // GS_R x 33: earlier vectors tile
  double* Bt = At + GS_R * 33;   // GS_R x 33: panel tile
  double* G = Bt + GS_R * 33;    // 32 x 33: G[c][p]
  double* red = G + GS_P * 33;   // 64
  for (int q = cs; q < ce; q += GS_P) {
    const int np = min(GS_P, ce - q);
    for (int rep = 0; rep < 2 && q > cs; ++rep) {
      for (int c0 = cs; c0 < q; c0 += 32) {
        const int nc = min(32, q - c0);
        // G = Z[:, c0:c0+nc]^T Z[:, q:q+np]; thread owns p = lane, c = 4*warp + i
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int r0 = 0; r0 < n; r0 += GS_R) {
          for (int e = tid; e < GS_R * 32; e += nt) {
            const int rr = e % GS_R, cc = e / GS_R, r = r0 + rr;
            At[rr * 33 + cc] = (r < n && cc < nc) ? Z[r + (long long)(c0 + cc) * ldz] : 0.0;
            Bt[rr * 33 + cc] = (r < n && cc < np) ? Z[r + (long long)(q + cc) * ldz] : 0.0;
          }
          __syncthreads();
#pragma unroll 8
          for (int rr = 0; rr < GS_R; ++rr) {
            const double bv = Bt[rr * 33 + lane];
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] += At[rr * 33 + 4 * warp + i] * bv;
          }
          __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) G[(4 * warp + i) * 33 + lane] = acc[i];
        __syncthreads();
        // Z[:, q+p] -= Z[:, c0:c0+nc] G[:, p]; thread per row
        for (int r = tid; r < n; r += nt) {
          double zp[GS_P];
#pragma unroll
          for (int p = 0; p < GS_P; ++p) zp[p] = p < np ? Z[r + (long long)(q + p) * ldz] : 0.0;
          for (int c = 0; c < nc; ++c) {
            const double z = Z[r + (long long)(c0 + c) * ldz];
#pragma unroll
            for (int p = 0; p < GS_P; ++p) zp[p] -= z * G[c * 33 + p];
          }
#pragma unroll
          for (int p = 0; p < GS_P; ++p)
            if (p < np) Z[r + (long long)(q + p) * ldz] = zp[p];
        }
        __syncthreads();
      }
    }
    // inside the panel: vector by vector
    for (int t = q; t < q + np; ++t) {
      double* zt = Z + (long long)t * ldz;
      for (int rep = 0; rep < 2 && t > q; ++rep) {
        for (int c = q + warp; c < t; c += nwarps) {
          const double* zc = Z + (long long)c * ldz;
          double s = 0.0;
          for (int r = lane; r < n; r += 32) s += zc[r] * zt[r];
          s = warp_sum(s);
          if (lane == 0) G[c - q] = s;
        }
        __syncthreads();
        for (int r = tid; r < n; r += nt) {
          double a = zt[r];
          for (int c = q; c < t; ++c) a -= G[c - q] * Z[r + (long long)c * ldz];
          zt[r] = a;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int r = tid; r < n; r += nt) part += zt[r] * zt[r];
      const double nrm2 = block_sum(part, red);
      const double sc = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
      for (int r = tid; r < n; r += nt) zt[r] *= sc;
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(256) k_band_mgs(const EigDev* __restrict__ jobs) {
  const EigDev J = jobs[blockIdx.x];
  const int kk = J.kk;
  __shared__ double sm[GS_SMEM_DOUBLES];
  for (int cs = 0; cs < kk;) {
    int ce = cs + 1;
    while (ce < kk && J.cstarts[ce] == cs) ++ce;
    if (ce - cs > 1) cluster_gs(J.Z, J.ldz, J.n, cs, ce, sm);
    cs = ce;
  }
}

// Zero the band rows of the reflector columns: V column j has its unit at
// row j + off (off = 1 one-stage, B2 two-stage).
__global__ void k_prep_v_off(const EigDev* __restrict__ jobs, int off) {
  const EigDev J = jobs[blockIdx.y];
  const int n = J.n;
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    if (i < j + off) J.A[i + j * J.lda] = 0.0;
    else if (i == j + off) J.A[i + j * J.lda] = 1.0;
  }
}

constexpr int kBlockedMinN = 128;

constexpr size_t kLatrdSmemMax = 200 * 1024;

template <int R>
void launch_latrd_t(Ctx& ctx, int count, int cs, size_t smem, const EigDev* dd, int j0) {
  smem_optin(k_latrd<R>, kLatrdSmemMax);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * cs);
  cfg.blockDim = dim3(LAT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ctx.launch_begin();
  HSVD_CUDA(cudaLaunchKernelEx(&cfg, k_latrd<R>, dd, j0, cs));
  ctx.check_launch("k_latrd");
}

void launch_latrd(Ctx& ctx, int R, int count, int cs, size_t smem, const EigDev* dd, int j0) {
  if (smem > kLatrdSmemMax) throw Error(kInvalid, "k_latrd: n too large");
  switch (R) {
    case 1: return launch_latrd_t<1>(ctx, count, cs, smem, dd, j0);
    case 2: return launch_latrd_t<2>(ctx, count, cs, smem, dd, j0);
    case 3: return launch_latrd_t<3>(ctx, count, cs, smem, dd, j0);
    case 4: return launch_latrd_t<4>(ctx, count, cs, smem, dd, j0);
    case 5: return launch_latrd_t<5>(ctx, count, cs, smem, dd, j0);
    case 6: return launch_latrd_t<6>(ctx, count, cs, smem, dd, j0);
    case 7:
    case 8: return launch_latrd_t<8>(ctx, count, cs, smem, dd, j0);
    case 9:
    case 10: return launch_latrd_t<10>(ctx, count, cs, smem, dd, j0);
    default:
      if (R <= 12) return launch_latrd_t<12>(ctx, count, cs, smem, dd, j0);
      throw Error(kInvalid, "k_latrd: n > 6144 not supported");
  }
}

// Reduction choice.  The two-stage path moves the O(n^3) work onto DMMA
// GEMMs but its band stages (panel QR, bulge chase, band inverse iteration)
// run one CTA (or a few) per matrix, so it pays off for large n or for
// batches that fill the GPU (measured on B200: single matrix, one-stage
// wins at n = 1024 and 2048, two-stage at 4096; 64 matrices of n = 2048,
// 2500 or 4096, two-stage wins).  HSVD_TWO_STAGE_MIN_N overrides with a
// plain size threshold.
constexpr int kTwoStageMinN = 1024;       // batched
constexpr int kTwoStageMinBatch = 32;
constexpr int kTwoStageAlwaysN = 3072;    // any batch size
bool use_two_stage(int nmax, int count) {
  if (const char* env = std::getenv("HSVD_TWO_STAGE_MIN_N")) return nmax >= std::atoi(env);
  return nmax >= kTwoStageAlwaysN || (nmax >= kTwoStageMinN && count >= kTwoStageMinBatch);
}

// Z <- Q Z with Q = H_0 H_1 ... (reflector of column j: unit at row j + off,
// stored in A column j), in compact-WY blocks of NBT reflectors.
void back_transform(Ctx& ctx, const std::vector<EigJob>& jobs, const std::vector<EigDev>& dev,
                    const EigDev* dd, int nmax, int off) {
  const int count = static_cast<int>(dev.size());
  if (nmax <= off + 1) return;
  const long long nn = (long long)nmax * nmax;
  int gx = static_cast<int>(std::min<long long>((nn + 255) / 256, 2048));
  ctx.launch_begin();
  k_prep_v_off<<<dim3(gx, count), 256, 0, ctx.stream>>>(dd, off);
  ctx.check_launch("k_prep_v");
  const int nblk_max = ceil_div(nmax - off, NBT);
  // S_b = V_b^T V_b for every block of every matrix (one grouped launch)
  std::vector<GemmDesc> ds;
  for (int g = 0; g < count; ++g) {
    const EigDev& e = dev[g];
    if (e.n <= off + 1) continue;
    for (int b = 0; b * NBT < e.n - off; ++b) {
      const int j0 = b * NBT, nb = std::min(NBT, e.n - off - j0), m = e.n - j0 - off;
      const double* V = e.A + j0 + off + (long long)j0 * e.lda;
      ds.push_back({V, V, e.S + (long long)b * NBT * NBT, e.lda, e.lda, NBT, nb, nb, m, 1.0, 0.0});
    }
  }
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, ds);
  const size_t tsm = ((size_t)NBT * (NBT + 1) + NBT) * sizeof(double);
  smem_optin(k_build_t, tsm);
  ctx.launch_begin();
  k_build_t<<<dim3(nblk_max, count), NBT, tsm, ctx.stream>>>(dd, off);
  ctx.check_launch("k_build_t");
  std::vector<double*> W(count), W2(count);
  for (int g = 0; g < count; ++g) {
    W[g] = ctx.arena.alloc_n<double>((size_t)NBT * jobs[g].kk);
    W2[g] = ctx.arena.alloc_n<double>((size_t)NBT * jobs[g].kk);
  }
  std::vector<GemmDesc> d1, d2, d3;
  for (int b = nblk_max - 1; b >= 0; --b) {
    const int j0 = b * NBT;
    d1.clear();
    d2.clear();
    d3.clear();
    for (int g = 0; g < count; ++g) {
      const EigDev& e = dev[g];
      const int nref = e.n - off;
      if (j0 >= nref || e.n <= off + 1) continue;
      const int m = e.n - j0 - off;
      const int nb = std::min(NBT, nref - j0);
      const double* V = e.A + j0 + off + (long long)j0 * e.lda;
      double* Zs = e.Z + j0 + off;
      d1.push_back({V, Zs, W[g], e.lda, e.ldz, NBT, nb, e.kk, m, 1.0, 0.0});  // W = V^T Zs
      d2.push_back({e.T + (long long)b * NBT * NBT, W[g], W2[g], NBT, NBT, NBT, nb, e.kk, nb, 1.0,
                    0.0});                                                    // W2 = T W
      d3.push_back({V, W2[g], Zs, e.lda, NBT, e.ldz, m, e.kk, nb, -1.0, 1.0});  // Zs -= V W2
    }
    if (d1.empty()) continue;
    gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, d1);
    gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, d2);
    gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, d3);
  }
}

// The job array is read by every launch of the solver, so it lives in arena
// memory rather than in the staging ring (which later launches recycle).
const EigDev* upload_jobs(Ctx& ctx, const std::vector<EigDev>& dev) {
  const size_t bytes = dev.size() * sizeof(EigDev);
  return static_cast<const EigDev*>(
      ctx.staging.put_to(ctx.arena.alloc(bytes), dev.data(), bytes, ctx.stream));
}

void two_stage(Ctx& ctx, const std::vector<EigJob>& jobs, std::vector<EigDev>& dev, int nmax,
               int kkmax) {
  const int count = static_cast<int>(dev.size());
  const int npan = ceil_div(nmax, B2);
  int kBandGroup = kBandGroupDefault;
  // eigenvectors: inverse iteration on the tridiagonal + the chase
  // reflectors (k_q2_apply), or inverse iteration on the band matrix
  // (k_band_invit).  Measured on B200 (64-matrix batches) with the on-chip
  // k_q2_apply: the first wins at n = 2048, 2500 and 4096 (1039 vs 1065 ms
  // at config 5 / 64 leaves).  HSVD_BAND_INVIT=1 forces the second.
  bool band_invit = nmax > kBandInvitMinN;
  if (const char* env = std::getenv("HSVD_BAND_INVIT")) band_invit = std::atoi(env) != 0;
  if (const char* env = std::getenv("HSVD_BAND_GROUP")) kBandGroup = std::max(1, std::atoi(env));
  size_t lu_slot_max = 0;
  for (int g = 0; g < count; ++g) {
    EigDev& d = dev[g];
    const int n = d.n;
    d.band = ctx.arena.alloc_n<double>((size_t)LDBB * n);
    d.band0 = band_invit ? ctx.arena.alloc_n<double>((size_t)LDBB * n) : nullptr;
    d.Tp = ctx.arena.alloc_n<double>((size_t)ceil_div(n, B2) * B2 * B2);
    d.psum = ctx.arena.alloc_n<double>((size_t)8 * B2 * B2);
    d.VW = ctx.arena.alloc_n<double>((size_t)n * 2 * B2 * kBandGroup);
    d.WV = ctx.arena.alloc_n<double>((size_t)n * 2 * B2 * kBandGroup);
    d.Y = ctx.arena.alloc_n<double>((size_t)n * B2);
    d.Z1 = ctx.arena.alloc_n<double>((size_t)2 * B2 * kBandGroup * B2);
    d.P1 = ctx.arena.alloc_n<double>((size_t)B2 * B2);
    d.Mb = ctx.arena.alloc_n<double>((size_t)B2 * B2);
    d.shifts = ctx.arena.alloc_n<double>(d.kk);
    d.cstarts = ctx.arena.alloc_n<int>(d.kk);
    d.vals_only = band_invit ? 1 : 2;
    if (!band_invit) {
      long long steps = 0;  // chase reflectors of all sweeps
      for (int s2 = 0; s2 <= n - 3; ++s2) steps += (n - 3 - s2) / B2 + 1;
      d.refl = ctx.arena.alloc_n<double>((size_t)std::max(1LL, steps) * (B2 + 1));
    }
    HSVD_CUDA(cudaMemsetAsync(d.band, 0, (size_t)LDBB * n * sizeof(double), ctx.stream));
    lu_slot_max = std::max(lu_slot_max, (size_t)n * (2 * B2 + 1 + B2 + 3));
  }
  // band LU workspaces (INV_WARPS slots per matrix; slot size of the largest n)
  // shifts spread over cpm CTAs per matrix (3 CTAs fit an SM), workspace
  // capped at 8 GB
  int cpm = std::max(1, std::min(ceil_div(3 * ctx.num_sms, count), ceil_div(kkmax, INV_WARPS)));
  while (cpm > 1 && lu_slot_max * sizeof(double) * INV_WARPS * cpm * count > (size_t(8) << 30)) --cpm;
  const int q2nc = std::max(1, q2_cols(nmax));
  const int q2x = ceil_div(kkmax, q2nc);
  if (band_invit) {
    double* lu = ctx.arena.alloc_n<double>(lu_slot_max * INV_WARPS * cpm * count);
    for (int g = 0; g < count; ++g) {  // indexed by blockIdx.x in the kernel
      dev[g].lu = lu;
      dev[g].lu_slot = (long long)lu_slot_max;
    }
  }
  const EigDev* dd = upload_jobs(ctx, dev);

  // stage 1: dense -> band.  The trailing update is delayed over groups of
  // kBandGroup panels: inside a group the panels' [V|W] pairs accumulate in
  // VW / WV (64 columns per panel), the next panel's columns and its
  // Y = A22 V are corrected with the pending pairs (small GEMMs with K = 64g),
  // and one SYR2K with K = 64 * kBandGroup updates the trailing matrix at the
  // end of the group (a quarter of the passes over A22).
  SubPhase sp1(ctx, "band");
  std::vector<GemmDesc> gc, g1, gz, gy, g2, g3, g4, g5, g6;
  for (int p = 0; p < npan; ++p) {
    const int j0 = p * B2, r0 = j0 + B2;
    const int gi = p % kBandGroup;        // panel index inside its group
    const int vcol = 2 * B2 * gi;         // its [V|W] columns in VW / WV
    const bool last_in_group = gi == kBandGroup - 1 || p == npan - 1;
    if (gi > 0) {  // columns j0..j0+B2 (rows j0..n) with the pending updates
      SubPhase sc(ctx, "band.corr");
      gc.clear();
      for (int g = 0; g < count; ++g) {
        const EigDev& e = dev[g];
        if (j0 >= e.n) continue;
        const int rows = e.n - j0, cols = std::min(B2, e.n - j0);
        gc.push_back({e.VW + j0, e.WV + j0, e.A + j0 + (long long)j0 * e.lda, e.n, e.n, e.lda, rows,
                      cols, vcol, -1.0, 1.0});
      }
      gemm_grouped(ctx, DType::F64, DType::F64, false, true, false, gc);
    }
    launch_panel_qr(ctx, count, std::max(0, nmax - r0), dd, j0, vcol);
    g1.clear(); gz.clear(); gy.clear(); g2.clear(); g3.clear(); g4.clear(); g5.clear(); g6.clear();
    for (int g = 0; g < count; ++g) {
      const EigDev& e = dev[g];
      const int n = e.n;
      if (r0 > n - 2) continue;
      const int m = n - r0;
      double* A22 = e.A + r0 + (long long)r0 * e.lda;
      const double* V = e.A + r0 + (long long)j0 * e.lda;
      const double* Tp = e.Tp + (long long)p * B2 * B2;
      double* X = e.VW + r0 + (long long)(vcol + B2) * n;
      g1.push_back({A22, V, e.Y + r0, e.lda, e.lda, n, m, B2, m, 1.0, 0.0});       // Y = A22 V
      if (gi > 0) {
        gz.push_back({e.WV + r0, V, e.Z1, n, e.lda, vcol, vcol, B2, m, 1.0, 0.0});  // Z1 = WV^T V
        gy.push_back({e.VW + r0, e.Z1, e.Y + r0, n, vcol, n, m, B2, vcol, -1.0, 1.0});  // Y -= VW Z1
      }
      g2.push_back({e.Y + r0, Tp, X, n, B2, n, m, B2, B2, 1.0, 0.0});               // X = Y T
      g3.push_back({V, X, e.P1, e.lda, n, B2, B2, B2, m, 1.0, 0.0});                // P1 = V^T X
      g4.push_back({Tp, e.P1, e.Mb, B2, B2, B2, B2, B2, B2, 1.0, 0.0});             // M = T^T P1
      g5.push_back({V, e.Mb, X, e.lda, B2, n, m, B2, B2, -0.5, 1.0});               // W = X - V M/2
      if (last_in_group)                                                             // syr2k
        g6.push_back({e.VW + r0, e.WV + r0, A22, n, n, e.lda, m, m, vcol + 2 * B2, -1.0, 1.0});
    }
    if (g1.empty()) {
      ctx.launch_begin();
      k_copy_w<<<dim3(1, count), 256, 0, ctx.stream>>>(dd, j0, vcol);
      ctx.check_launch("k_copy_w");
      continue;
    }
    {
      SubPhase sy(ctx, "band.y");
      gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, g1);
      if (!gz.empty()) {
        gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, gz);
        gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, gy);
      }
    }
    {
      SubPhase sw(ctx, "band.w");
      gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, g2);
      gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, g3);
      gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, g4);
      gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, g5);
      ctx.launch_begin();
      k_copy_w<<<dim3(256, count), 256, 0, ctx.stream>>>(dd, j0, vcol);
      ctx.check_launch("k_copy_w");
    }
    if (!g6.empty()) {
      SubPhase s2k(ctx, "band.syr2k");
      gemm_grouped(ctx, DType::F64, DType::F64, false, true, true, g6);
    }
  }
  if (band_invit)  // the band before the chase, for the band inverse iteration
    for (int g = 0; g < count; ++g)
      HSVD_CUDA(cudaMemcpyAsync(dev[g].band0, dev[g].band, (size_t)LDBB * dev[g].n * sizeof(double),
                                cudaMemcpyDeviceToDevice, ctx.stream));
  // stage 2: band -> tridiagonal (values), eigenvalues by bisection
  SubPhase sp2(ctx, "tri");
  ctx.launch_begin();
  // spread each matrix's sweeps over a cluster while SMs would idle
  int ccs = 1;
  while (ccs < 2 && count * ccs * 2 <= ctx.num_sms) ccs *= 2;  // 4 measured slower
  if (const char* env = std::getenv("HSVD_CHASE_CS")) ccs = std::max(1, std::atoi(env));
  if (ccs == 1) {
    k_chase<false><<<count, CHASE_WARPS * 32, 0, ctx.stream>>>(dd, 1);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(count * ccs);
    cfg.blockDim = dim3(CHASE_WARPS * 32);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = ctx.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = ccs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    HSVD_CUDA(cudaLaunchKernelEx(&cfg, k_chase<true>, dd, ccs));
  }
  ctx.check_launch("k_chase");
  {
    const size_t smem = (3 * (size_t)nmax + 3 * (size_t)kkmax + 32) * sizeof(double) +
                        (size_t)std::max(kkmax, EIG_THREADS) * sizeof(int) + 64;
    smem_optin(k_steig, smem);
    ctx.launch_begin();
    k_steig<<<count, EIG_THREADS, smem, ctx.stream>>>(dd);
    ctx.check_launch("k_steig");
  }
  // eigenvectors of the band matrix
  if (!band_invit) {
    ctx.launch_begin();
    k_band_mgs<<<count, 256, 0, ctx.stream>>>(dd);  // clusters of the tridiagonal's vectors
    ctx.check_launch("k_band_mgs");
    ctx.launch_begin();
    const size_t q2smem = q2_smem(nmax, q2nc);
    if (q2nc == 8) {
      smem_optin(k_q2_apply<8>, q2smem);
      k_q2_apply<8><<<dim3(q2x, count), Q2_WARPS * 32, q2smem, ctx.stream>>>(dd);
    } else if (q2nc == 4) {
      smem_optin(k_q2_apply<4>, q2smem);
      k_q2_apply<4><<<dim3(q2x, count), Q2_WARPS * 32, q2smem, ctx.stream>>>(dd);
    } else {
      smem_optin(k_q2_apply<2>, q2smem);
      k_q2_apply<2><<<dim3(q2x, count), Q2_WARPS * 32, q2smem, ctx.stream>>>(dd);
    }
    ctx.check_launch("k_q2_apply");
  } else {
    const size_t smem =
        ((size_t)INV_WARPS * ((B2 + 1) * (2 * B2 + 1) + INV_RING) + 64) * sizeof(double);
    smem_optin(k_band_invit, smem);
    ctx.launch_begin();
    k_band_invit<<<dim3(cpm, count), INV_WARPS * 32, smem, ctx.stream>>>(dd);
    ctx.check_launch("k_band_invit");
    ctx.launch_begin();
    k_band_mgs<<<count, 256, 0, ctx.stream>>>(dd);
    ctx.check_launch("k_band_mgs");
  }
  // back through the stage-1 reflectors
  SubPhase sp3(ctx, "back");
  back_transform(ctx, jobs, dev, dd, nmax, B2);
}

}  // namespace

void eig_topk(Ctx& ctx, const std::vector<EigJob>& jobs_in) {
  std::vector<EigJob> jobs;
  for (const auto& j : jobs_in)
    if (j.n > 0 && j.kk > 0) jobs.push_back(j);
  if (jobs.empty()) return;
  const int count = static_cast<int>(jobs.size());
  Arena::Mark mk = ctx.arena.mark();
  std::vector<EigDev> dev(count);
  int nmax = 0, kkmax = 0;
  const bool inline_gs =
      std::getenv("HSVD_STEIG_INLINE_GS") && std::atoi(std::getenv("HSVD_STEIG_INLINE_GS")) != 0;
  for (int g = 0; g < count; ++g) {
    const EigJob& j = jobs[g];
    if (j.kk > j.n) throw Error(kInvalid, "eig_topk: kk > n");
    if (j.n > 6144) throw Error(kInvalid, "eig_topk: n > 6144 not supported");
    EigDev& d = dev[g];
    d.A = j.A;
    d.lda = j.lda;
    d.n = j.n;
    d.kk = j.kk;
    d.d = ctx.arena.alloc_n<double>(j.n);
    d.e = ctx.arena.alloc_n<double>(j.n);
    d.tau = ctx.arena.alloc_n<double>(j.n);
    d.lam = j.lam;
    d.Z = j.Z;
    d.ldz = j.ldz;
    d.piv = ctx.arena.alloc_n<double>((size_t)j.n * j.kk);
    // inverse iteration without the in-iteration Gram-Schmidt; clusters are
    // orthonormalised once afterwards by the blocked k_band_mgs
    // (HSVD_STEIG_INLINE_GS=1: dstein's per-iteration MGS inside k_steig)
    d.shifts = ctx.arena.alloc_n<double>(j.kk);
    d.cstarts = ctx.arena.alloc_n<int>(j.kk);
    d.vals_only = inline_gs ? 0 : 2;
    const int nblk = std::max(1, ceil_div(j.n - 1, NBT));
    d.T = ctx.arena.alloc_n<double>((size_t)nblk * NBT * NBT);
    d.S = ctx.arena.alloc_n<double>((size_t)nblk * NBT * NBT);
    nmax = std::max(nmax, j.n);
    kkmax = std::max(kkmax, j.kk);
  }
  const EigDev* dd = upload_jobs(ctx, dev);

  if (use_two_stage(nmax, count)) {
    two_stage(ctx, jobs, dev, nmax, kkmax);
    ctx.arena.release(mk);
    return;
  }
  // 1. tridiagonalise
  int blocked_min = kBlockedMinN;
  if (const char* env = std::getenv("HSVD_BLOCKED_MIN_N")) blocked_min = std::atoi(env);
  if (nmax >= blocked_min) {
    for (int g = 0; g < count; ++g) {
      dev[g].VW = ctx.arena.alloc_n<double>((size_t)dev[g].n * 2 * NB);
      dev[g].WV = ctx.arena.alloc_n<double>((size_t)dev[g].n * 2 * NB);
    }
    dd = upload_jobs(ctx, dev);
    const int R = ceil_div(nmax, LAT);
    // cluster size: spread each matrix's mat-vec over several SMs while the
    // batch alone would leave SMs idle (portable cluster size <= 8)
    int cs = 1;
    while (cs < 8 && (long long)count * cs * 2 <= ctx.num_sms &&
           ((size_t)nmax * (1 + 4 * cs) + 4 * NB + 64) * sizeof(double) <= kLatrdSmemMax)
      cs *= 2;
    if (const char* env = std::getenv("HSVD_LATRD_CS")) cs = std::max(1, std::atoi(env));
    const size_t smem = ((size_t)nmax * (1 + 2 * cs) + 4 * NB + 64) * sizeof(double);
    std::vector<GemmDesc> upd;
    for (int j0 = 0; j0 < nmax - 1; j0 += NB) {
      launch_latrd(ctx, R, count, cs, smem, dd, j0);
      upd.clear();
      for (int g = 0; g < count; ++g) {
        const EigDev& e = dev[g];
        const int nref = e.n - 1;
        if (e.n <= 2 || j0 + NB >= nref) continue;
        const int j1 = j0 + NB, m = e.n - j1;
        upd.push_back({e.VW + j1, e.WV + j1, e.A + j1 + (long long)j1 * e.lda, e.n, e.n, e.lda, m,
                       m, 2 * NB, -1.0, 1.0});
      }
      // A22 -= [V W] [W V]^T  (symmetric: lower tiles + mirror)
      gemm_grouped(ctx, DType::F64, DType::F64, false, true, true, upd);
    }
  } else {
    const size_t smem = (4 * (size_t)nmax + TRD_THREADS + 64) * sizeof(double);
    smem_optin(k_sytrd, smem);
    ctx.launch_begin();
    k_sytrd<<<count, TRD_THREADS, smem, ctx.stream>>>(dd);
    ctx.check_launch("k_sytrd");
  }
  // 2. tridiagonal eigenpairs
  {
    const size_t smem = (3 * (size_t)nmax + 3 * (size_t)kkmax + 32) * sizeof(double) +
                        (size_t)std::max(kkmax, EIG_THREADS) * sizeof(int) + 64;
    smem_optin(k_steig, smem);
    ctx.launch_begin();
    k_steig<<<count, EIG_THREADS, smem, ctx.stream>>>(dd);
    ctx.check_launch("k_steig");
    if (!inline_gs) {
      ctx.launch_begin();
      k_band_mgs<<<count, 256, 0, ctx.stream>>>(dd);
      ctx.check_launch("k_band_mgs");
    }
  }
  // 3. back-transform Z <- Q Z (blocks applied last to first)
  back_transform(ctx, jobs, dev, dd, nmax, 1);
  ctx.arena.release(mk);
}

}  // namespace hsvdcu
