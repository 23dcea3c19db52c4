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
//   (two-stage reduction for large n: syev_band.cu)
#include "syev_impl.cuh"

namespace hsvdcu {
namespace syev_impl {

namespace {

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
      // columns per batch: loads in flight per thread (R rows each)
      constexpr int U = R == 1 ? 24 : R == 2 ? 12 : (R <= 3) ? 8 : (R <= 6 ? 6 : 3);
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

// The same count with q_{i-1}^-1 from the hardware reciprocal seed refined
// by Newton steps instead of the IEEE division sequence: each operation
// still carries a relative error of a few ulps, which is all the backward
// stability of the Sturm count needs (Kahan; dstebz's analysis).
__device__ __forceinline__ double fast_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  double e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  e = fma(-q, r, 1.0);
  r = fma(r, e, r);
  return r;
}
__device__ __forceinline__ int sturm_count_less_rcp(const double* dd, const double* e2, int n,
                                                    double x, double pivmin) {
  double q = dd[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int cnt = q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = (dd[i] - x) - e2[i - 1] * fast_rcp(q);
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}


__global__ void __launch_bounds__(EIG_THREADS) k_steig(const EigDev* __restrict__ jobs, int pforce,
                                                       int flags) {
  const EigDev J = jobs[blockIdx.x];
  const int n = J.n, kk = J.kk;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
  extern __shared__ double sm[];
  // the tridiagonal and the per-eigenvalue arrays live in shared memory, or
  // (large n or kk) in global scratch (3n + 3kk doubles)
  double* dd = J.trig ? J.trig : sm;
  double* ee = dd + n;
  double* e2 = ee + n;
  double* lam = e2 + n;
  double* shift = lam + kk;
  double* dots = shift + kk;
  double* red = J.trig ? sm : dots + kk;
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
    const int P = max(1, pforce > 0 ? min(pforce, nt / kk) : nt / kk);
    const bool rcpc = flags & 1;
    // flags & 2: dstebz's criterion with ABSTOL <= 0 -- converged once the
    // bracket is below max(ulp |T|, 2 ulp |lambda|) -- instead of relative
    // accuracy for every eigenvalue (experiment only, see launch_steig)
    const double atol = (flags & 2) ? eps * tnorm : 0.0;
    auto count = [&](double x) {
      return rcpc ? sturm_count_less_rcp(dd, e2, n, x, pivmin) : sturm_count_less(dd, e2, n, x, pivmin);
    };
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
          const double tol = fmax(atol, 2.0 * eps * fmax(fabs(lo), fabs(hi))) + 4.0 * pivmin;
          if (hi - lo <= tol) break;
          const double mid = 0.5 * (lo + hi);
          if (mid <= lo || mid >= hi) break;
          if (count(mid) > idx) hi = mid;
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
          const double tol = fmax(atol, 2.0 * eps * fmax(fabs(lo), fabs(hi))) + 4.0 * pivmin;
          x = lo + (hi - lo) * (double)(g + 1) / (double)(P + 1);
          active = hi - lo > tol && x > lo && x < hi;
          cnt[t * P + g] = active ? count(x) : -1;
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
  const bool rcpi = flags & 4;  // the solves' divisions through fast_rcp too
  // The iterates and pivots live in the scratch J.piv in row-major [n][kk]
  // layout: thread t walks its vector row by row, so a warp's accesses to
  // one row are coalesced.  They stream through registers IC rows at a time,
  // the next chunk's loads issued before the current chunk's recurrence.
  constexpr int IC = 8;
  const long long nk = (long long)n * kk;
  double* const Dt = J.piv;       // pivots of L D L^T = T - shift_t I (column t)
  double* const Zt = J.piv + nk;  // iterates
  // start vectors (deterministic pseudo-random, dstein uses dlarnv uniform(-1,1))
  for (long long e = tid; e < nk; e += nt) {
    const int r = (int)(e / kk), t = (int)(e % kk);
    const unsigned h = hash32((unsigned)r * 2654435761u ^ hash32((unsigned)t + 0x9e3779b9u));
    Zt[e] = ((double)h / 4294967296.0) * 2.0 - 1.0;
  }
  __syncthreads();

  for (int it = 0; it < 3; ++it) {
    for (int t = tid; t < kk; t += nt) {
      const double s = shift[t];
      double* z = Zt + t;  // row r at z[r * kk]
      double* Dw = Dt + t;
      auto at = [&](int r) { return (long long)r * kk; };
      double D = guard_pivot(dd[0] - s, tiny);
      Dw[0] = D;
      double y = z[0];
      double nz[IC], nd[IC];
#pragma unroll
      for (int j = 0; j < IC; ++j) nz[j] = 1 + j < n ? z[at(1 + j)] : 0.0;
      for (int r0 = 1; r0 < n; r0 += IC) {
        double cz[IC], cd[IC];
#pragma unroll
        for (int j = 0; j < IC; ++j) cz[j] = nz[j];
#pragma unroll
        for (int j = 0; j < IC; ++j) nz[j] = r0 + IC + j < n ? z[at(r0 + IC + j)] : 0.0;
#pragma unroll
        for (int j = 0; j < IC; ++j) {
          const int r = r0 + j;
          if (r < n) {
            const double l = rcpi ? ee[r - 1] * fast_rcp(D) : ee[r - 1] / D;
            D = guard_pivot(dd[r] - s - l * ee[r - 1], tiny);
            cd[j] = D;
            y = cz[j] - l * y;
            cz[j] = y;
          }
        }
#pragma unroll
        for (int j = 0; j < IC; ++j)
          if (r0 + j < n) {
            z[at(r0 + j)] = cz[j];
            Dw[at(r0 + j)] = cd[j];
          }
      }
      double zr = z[at(n - 1)] / Dw[at(n - 1)];
      z[at(n - 1)] = zr;
      double nrm2 = zr * zr;
#pragma unroll
      for (int j = 0; j < IC; ++j) {
        nz[j] = n - 2 - j >= 0 ? z[at(n - 2 - j)] : 0.0;
        nd[j] = n - 2 - j >= 0 ? Dw[at(n - 2 - j)] : 1.0;
      }
      for (int r0 = n - 2; r0 >= 0; r0 -= IC) {
        double cz[IC], cd[IC];
#pragma unroll
        for (int j = 0; j < IC; ++j) {
          cz[j] = nz[j];
          cd[j] = nd[j];
        }
#pragma unroll
        for (int j = 0; j < IC; ++j) {
          const int r = r0 - IC - j;
          nz[j] = r >= 0 ? z[at(r)] : 0.0;
          nd[j] = r >= 0 ? Dw[at(r)] : 1.0;
        }
#pragma unroll
        for (int j = 0; j < IC; ++j) {
          const int r = r0 - j;
          if (r >= 0) {
            zr = rcpi ? (cz[j] - ee[r] * zr) * fast_rcp(cd[j]) : (cz[j] - ee[r] * zr) / cd[j];
            cz[j] = zr;
            nrm2 += zr * zr;
          }
        }
#pragma unroll
        for (int j = 0; j < IC; ++j)
          if (r0 - j >= 0) z[at(r0 - j)] = cz[j];
      }
      double sc = 1.0 / sqrt(nrm2);
      if (!isfinite(sc) || nrm2 == 0.0) sc = 0.0;
      for (int r0 = 0; r0 < n; r0 += IC) {
        double cz[IC];
#pragma unroll
        for (int j = 0; j < IC; ++j) cz[j] = r0 + j < n ? z[at(r0 + j)] : 0.0;
#pragma unroll
        for (int j = 0; j < IC; ++j)
          if (r0 + j < n) z[at(r0 + j)] = cz[j] * sc;
      }
      if (sc == 0.0) z[at(t % n)] = 1.0;
    }
    __syncthreads();
    if (it == 0 || J.vals_only == 2) continue;
    // Gram-Schmidt (twice) inside clusters, in eigenvalue order
    for (int t = 0; t < kk; ++t) {
      const int cs = cstart[t];
      if (cs == t) continue;
      double* zt = Zt + t;
      for (int rep = 0; rep < 2; ++rep) {
        for (int c = cs + warp; c < t; c += nwarps) {
          const double* zc = Zt + c;
          double s = 0.0;
          for (int r = lane; r < n; r += 32) s += zc[(long long)r * kk] * zt[(long long)r * kk];
          s = warp_sum(s);
          if (lane == 0) dots[c - cs] = s;
        }
        __syncthreads();
        for (int r = tid; r < n; r += nt) {
          double a = zt[(long long)r * kk];
          for (int c = cs; c < t; ++c) a -= dots[c - cs] * Zt[(long long)r * kk + c];
          zt[(long long)r * kk] = a;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int r = tid; r < n; r += nt) part += zt[(long long)r * kk] * zt[(long long)r * kk];
      const double nrm2 = block_sum(part, red);
      const double sc = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
      for (int r = tid; r < n; r += nt) zt[(long long)r * kk] *= sc;
      __syncthreads();
    }
  }
  // iterates -> Z (column-major), R rows at a time through shared memory
  // (the tridiagonal's dd, ee, e2 are dead: 3n doubles)
  {
    double* stage = dd;
    const int R = max(1, min(n, 3 * n / kk));
    for (int r0 = 0; r0 < n; r0 += R) {
      const int rows = min(R, n - r0);
      for (int e = tid; e < rows * kk; e += nt) stage[e] = Zt[(long long)r0 * kk + e];
      __syncthreads();
      for (int e = tid; e < rows * kk; e += nt) {
        const int i = e % rows, t = e / rows;
        J.Z[(long long)t * J.ldz + r0 + i] = stage[i * kk + t];
      }
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

// One panel of a large cluster (k_gs_panel): its vectors orthonormalised
// among themselves after the GEMM projections against the cluster's earlier
// panels (launch_band_mgs).
struct GsPanel {
  double* Z;
  long long ldz;
  int n, q, np;
};

__global__ void __launch_bounds__(256, 2) k_gs_panel(const GsPanel* __restrict__ pan) {
  const GsPanel P = pan[blockIdx.x];
  __shared__ double sm[GS_SMEM_DOUBLES];
  cluster_gs(P.Z, P.ldz, P.n, P.q, P.q + P.np, sm);
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
// batches that fill the GPU.  Measured on B200 (round 2, after the chase and
// Q2 improvements of round 1; profiles/r02_eig_batch*.json, top-kk device
// time): two-stage wins at n >= 2048 for every batch size -- 1 x 2048: 65 vs
// 77 ms, 8 x 2048: 67 vs 106, 8 x 2500: 91 vs 216, 2 x 4096: 184 vs 1151 --
// so the per-rank leaf batches of a multi-GPU run (8 leaves per rank at 8
// GPUs for configs 2-4) keep the two-stage path; one-stage still wins at
// n = 1024 and 1536 for small batches (17 vs 28 ms, 41 vs 45 ms).
// HSVD_TWO_STAGE_MIN_N overrides with a plain size threshold.
constexpr int kTwoStageMinN = 1024;       // batched
constexpr int kTwoStageMinBatch = 32;
constexpr int kTwoStageAlwaysN = 2048;    // any batch size
bool use_two_stage(int nmax, int count) {
  if (const char* env = std::getenv("HSVD_TWO_STAGE_MIN_N")) return nmax >= std::atoi(env);
  return nmax >= kTwoStageAlwaysN || (nmax >= kTwoStageMinN && count >= kTwoStageMinBatch);
}

}  // namespace

// Z <- Q Z with Q = H_0 H_1 ... (reflector of column j: unit at row j + off,
// stored in A column j), in compact-WY blocks of NBT reflectors.
// The reflector-only part of the back-transform (explicit V, S = V^T V and
// the T factors of the WY blocks): independent of the eigenvectors, so the
// two-stage driver runs it on the side stream under the bulge chase.
void back_prepare(Ctx& ctx, const std::vector<EigDev>& dev, const EigDev* dd, int nmax, int off) {
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
}

// Z <- Q Z through the WY blocks prepared by back_prepare (last block first).
void back_apply(Ctx& ctx, const std::vector<EigJob>& jobs, const std::vector<EigDev>& dev,
                int nmax, int off) {
  const int count = static_cast<int>(dev.size());
  if (nmax <= off + 1) return;
  const int nblk_max = ceil_div(nmax - off, NBT);
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

void back_transform(Ctx& ctx, const std::vector<EigJob>& jobs, const std::vector<EigDev>& dev,
                    const EigDev* dd, int nmax, int off) {
  back_prepare(ctx, dev, dd, nmax, off);
  back_apply(ctx, jobs, dev, nmax, off);
}

// The job array is read by every launch of the solver, so it lives in arena
// memory rather than in the staging ring (which later launches recycle).
const EigDev* upload_jobs(Ctx& ctx, const std::vector<EigDev>& dev) {
  const size_t bytes = dev.size() * sizeof(EigDev);
  return static_cast<const EigDev*>(
      ctx.staging.put_to(ctx.arena.alloc(bytes), dev.data(), bytes, ctx.stream));
}

constexpr size_t kSteigSmemMax = 220 * 1024;
size_t steig_smem(int nmax, int kkmax, bool global_tri) {
  return ((global_tri ? 0 : 3 * (size_t)nmax + 3 * (size_t)kkmax) + 32) * sizeof(double) +
         (size_t)std::max(kkmax, EIG_THREADS) * sizeof(int) + 64;
}
bool steig_global_tri(int nmax, int kkmax) { return steig_smem(nmax, kkmax, false) > kSteigSmemMax; }

void launch_steig(Ctx& ctx, const EigDev* dd, int count, int nmax, int kkmax) {
    const size_t smem = steig_smem(nmax, kkmax, steig_global_tri(nmax, kkmax));
    smem_optin(k_steig, smem);
    ctx.launch_begin();
    // flags: 1 Sturm counts through fast_rcp, 4 the inverse-iteration solves
    // through fast_rcp (measured round 2: config 5 k_steig 49.5 + 19.7 ->
    // 34.0 + 13.3 ms with 1; P = 1 bisection instead of the 2-point
    // multisection was slower: 62.8 + 25.6 ms).  2, dstebz's absolute
    // tolerance ulp |T| (30.0 + 11.1 ms), is not used: the retained tail of a
    // leaf can hold eigenvalues ~1e-14 |T| whose shifts then lose the digits
    // inverse iteration needs to separate them (config-5 stand-in: sigma off
    // by 1.5e-3 against the oracle).
    int pforce = 0, flags = 5;
    if (const char* e = std::getenv("HSVD_STEIG_P")) pforce = std::atoi(e);
    if (const char* e = std::getenv("HSVD_STEIG_FLAGS")) flags = std::atoi(e);
    k_steig<<<count, EIG_THREADS, smem, ctx.stream>>>(dd, pforce, flags);
    ctx.check_launch("k_steig");
}

// Clusters of at least kBigCluster vectors (many eigenpairs requested, e.g.
// the whole spectrum of a block under the default MatConfig, where dstein's
// 1e-3 |T| rule groups most of them) would cost one CTA O(n c^2) in
// k_band_mgs; they are orthonormalised instead by block classical
// Gram-Schmidt twice over panels of GS_PW vectors, the projections against
// the cluster's earlier panels as grouped DMMA GEMMs across the GPU and each
// panel's own vectors by k_gs_panel.  The cluster starts are read back to
// plan that (one small device->host copy, only when kk >= kBigCluster); big
// clusters are then marked as singletons for k_band_mgs.
constexpr int kBigClusterDefault = 96;  // measured: config 5 k_band_mgs 24.1 -> 11.0 + GEMMs (64 leaves) with 96..128 against 192
constexpr int GS_PW = 64;

void launch_band_mgs(Ctx& ctx, const EigDev* dd, const std::vector<EigDev>& dev) {
  const int count = static_cast<int>(dev.size());
  struct Big {
    int g, cs, ce;
    double* W;
  };
  std::vector<Big> big;
  int kkmax = 0;
  for (const EigDev& e : dev) kkmax = std::max(kkmax, e.kk);
  int kBigCluster = kBigClusterDefault;
  if (const char* env = std::getenv("HSVD_BIG_CLUSTER")) kBigCluster = std::max(GS_PW, std::atoi(env));
  if (kkmax >= kBigCluster) {
    std::vector<size_t> off(count + 1, 0);
    for (int g = 0; g < count; ++g) off[g + 1] = off[g] + dev[g].kk;
    int* h = ctx.pinned_ints(off[count]);
    for (int g = 0; g < count; ++g)
      HSVD_CUDA(cudaMemcpyAsync(h + off[g], dev[g].cstarts, dev[g].kk * sizeof(int),
                                cudaMemcpyDeviceToHost, ctx.stream));
    HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
    std::vector<int> hc(h, h + off[count]);
    for (int g = 0; g < count; ++g) {
      const int kk = dev[g].kk;
      int* c = hc.data() + off[g];
      bool changed = false;
      for (int cs = 0; cs < kk;) {
        int ce = cs + 1;
        while (ce < kk && c[ce] == cs) ++ce;
        if (ce - cs >= kBigCluster) {
          big.push_back({g, cs, ce, ctx.arena.alloc_n<double>((size_t)(ce - cs) * GS_PW)});
          for (int i = cs; i < ce; ++i) c[i] = i;  // singletons for k_band_mgs
          changed = true;
        }
        cs = ce;
      }
      if (changed)
        ctx.staging.put_to(dev[g].cstarts, c, kk * sizeof(int), ctx.stream);
    }
  }
  ctx.launch_begin();
  k_band_mgs<<<count, 256, 0, ctx.stream>>>(dd);
  ctx.check_launch("k_band_mgs");
  if (big.empty()) return;
  int npan = 0;
  for (const Big& b : big) npan = std::max(npan, ceil_div(b.ce - b.cs, GS_PW));
  std::vector<GemmDesc> d1, d2;
  std::vector<GsPanel> pans;
  for (int j = 0; j < npan; ++j) {
    d1.clear();
    d2.clear();
    pans.clear();
    for (const Big& b : big) {
      const int q = b.cs + j * GS_PW;
      if (q >= b.ce) continue;
      const EigDev& e = dev[b.g];
      const int np = std::min(GS_PW, b.ce - q), M = q - b.cs;
      double* Zp = e.Z + (long long)q * e.ldz;
      const double* Zc = e.Z + (long long)b.cs * e.ldz;
      if (M > 0) {
        d1.push_back({Zc, Zp, b.W, e.ldz, e.ldz, M, M, np, e.n, 1.0, 0.0});    // W = Zc^T Zp
        d2.push_back({Zc, b.W, Zp, e.ldz, M, e.ldz, e.n, np, M, -1.0, 1.0});  // Zp -= Zc W
      }
      pans.push_back({e.Z, e.ldz, e.n, q, np});
    }
    for (int rep = 0; rep < 2 && !d1.empty(); ++rep) {
      gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, d1);
      gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, d2);
    }
    const size_t bytes = pans.size() * sizeof(GsPanel);
    const GsPanel* dp = static_cast<const GsPanel*>(
        ctx.staging.put_to(ctx.arena.alloc(bytes), pans.data(), bytes, ctx.stream));
    ctx.launch_begin();
    k_gs_panel<<<(unsigned)pans.size(), 256, 0, ctx.stream>>>(dp);
    ctx.check_launch("k_gs_panel");
  }
}

}  // namespace syev_impl

void eig_topk(Ctx& ctx, const std::vector<EigJob>& jobs_in) {
  using namespace syev_impl;
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
    d.piv = ctx.arena.alloc_n<double>((size_t)2 * j.n * j.kk);  // k_steig: pivots + iterates
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
  if (steig_global_tri(nmax, kkmax))  // k_steig's tridiagonal in global memory
    for (int g = 0; g < count; ++g)
      dev[g].trig = ctx.arena.alloc_n<double>((size_t)3 * dev[g].n + 3 * (size_t)dev[g].kk);
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
    launch_steig(ctx, dd, count, nmax, kkmax);
    if (!inline_gs) {
      launch_band_mgs(ctx, dd, dev);
    }
  }
  // 3. back-transform Z <- Q Z (blocks applied last to first)
  back_transform(ctx, jobs, dev, dd, nmax, 1);
  ctx.arena.release(mk);
}

}  // namespace hsvdcu
