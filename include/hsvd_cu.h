/*
 * hsvd_cu.h -- C ABI of the B200-native hierarchical merge-and-truncate SVD.
 *
 * Drop-in boundary for the hot path of the reference library hsvd::core
 * (/root/reference/proj/core).  The reference has no FFI; its boundary is the
 * C++ API below, and each entry point here replaces one of those functions
 * (same argument meaning, same error behaviour mapped to status codes):
 *
 *   hsvd_cu_hierarchical_svd     hsvd::hierarchical_svd      hierarchy.hpp:45, hierarchy.cpp:65-94
 *   hsvd_cu_recover_left_vectors hsvd::recover_left_vectors  hierarchy.hpp:50, hierarchy.cpp:96-112
 *   hsvd_cu_rank_k_svd           hierarchical_svd followed by recover_left_vectors
 *                                (the pipeline of hsvd_main.cpp:132-143 / bench.cpp:109-113)
 *   hsvd_cu_svd_of_col_slices    hsvd::svd_of_col_slices     hierarchy.hpp:39-40, hierarchy.cpp:50-63
 *   hsvd_cu_tree_merge           hsvd::tree_merge            hierarchy.hpp:32-34, hierarchy.cpp:31-48
 *   hsvd_cu_merge_pair           hsvd::merge_pair_qr /       merge.hpp:19-30, merge.cpp:42-117
 *                                hsvd::merge_pair_naive
 *   hsvd_cu_full_svd             hsvd::full_svd              kernels.hpp:26, kernels.cpp:21-48
 *   hsvd_cu_qr_thin              hsvd::qr_thin               kernels.hpp:29, kernels.cpp:50-61
 *   hsvd_cu_refine_factors       hsvd::refine_factors        refine.hpp:18-21, refine.cpp:26-72
 *
 * Matrices crossing the boundary use the reference's DenseMatrix layout:
 * row-major, real64 (fp32 is accepted for the input matrix X), leading
 * dimension in elements.  Results live in device memory owned by the context
 * and are valid until the next call on the same context; the accessors copy
 * them out (row-major) or expose the column-major device pointers.
 *
 * Every function returns HSVD_CU_OK or an error code; hsvd_cu_last_error()
 * returns the thread-local message (HSVD_CU_EINVAL <-> std::invalid_argument,
 * HSVD_CU_EDECOMP <-> hsvd::DecompositionError with rows/cols from
 * hsvd_cu_last_error_dims(), HSVD_CU_EIO / HSVD_CU_EFORMAT <-> hsvd::IoError /
 * hsvd::FormatError of the matrix loader).  There is no CPU fallback: without a CUDA
 * device every compute entry point fails with HSVD_CU_ECUDA.
 */
#ifndef HSVD_CU_H_
#define HSVD_CU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hsvd_cu_ctx hsvd_cu_ctx;
typedef struct hsvd_cu_result hsvd_cu_result;

enum {
  HSVD_CU_OK = 0,
  HSVD_CU_EINVAL = 1,
  HSVD_CU_EDECOMP = 2,
  HSVD_CU_ECUDA = 3,
  HSVD_CU_ENCCL = 4,
  HSVD_CU_ENOMEM = 5,
  HSVD_CU_EIO = 6,     /* hsvd::IoError (matrix_io.hpp) */
  HSVD_CU_EFORMAT = 7  /* hsvd::FormatError (matrix_io.hpp) */
};
enum { HSVD_CU_F32 = 0, HSVD_CU_F64 = 1 };
enum { HSVD_CU_COLUMN_CONCAT = 0, HSVD_CU_ROW_CONCAT = 1 };
enum { HSVD_CU_HOST = 0, HSVD_CU_DEVICE = 1 };

/* hsvd::MatConfig (svd_factor.hpp:28-35); max_rank <= 0 means "no cap". */
typedef struct {
  double gamma;
  int64_t row_block_rows;
  int64_t col_block_cols;
  double epsilon;
  int32_t max_iters;
  int64_t max_rank;
} hsvd_cu_config;

/* One side of an hsvd::SvdFactor (svd_factor.hpp:14-25): the carried basis
 * (dim x rank, row-major, leading dimension ld, host memory) and sigma. */
typedef struct {
  const double* basis;
  int64_t dim;
  int64_t rank;
  int64_t ld;
  const double* sigma;
  int32_t degenerate;
} hsvd_cu_factor_in;

int hsvd_cu_version(void);
const char* hsvd_cu_last_error(void);
void hsvd_cu_last_error_dims(int64_t* rows, int64_t* cols);

int hsvd_cu_ctx_create(int device, hsvd_cu_ctx** out);
int hsvd_cu_ctx_destroy(hsvd_cu_ctx* ctx);
/* cudaStream_t the context launches on (for event timing by callers). */
int hsvd_cu_ctx_stream(hsvd_cu_ctx* ctx, void** stream);
/* Number of kernels this library has launched on the context. */
int64_t hsvd_cu_launch_count(const hsvd_cu_ctx* ctx);
/* Device bytes currently reserved by the context arena. */
int64_t hsvd_cu_arena_bytes(const hsvd_cu_ctx* ctx);
int hsvd_cu_synchronize(hsvd_cu_ctx* ctx);
/* Per-launch CUDA-event timing of this library's kernels (for benchmarks).
 * report: "phase[/sub]:kernel\tlaunches\ttotal_ms\tflops\tbytes\n" lines
 * since the last report (flops: algorithmic flops of the GEMM launches, else
 * 0; bytes: algorithmic HBM bytes of the factor-streaming launches, else 0);
 * returns the bytes needed (including the NUL), or -1 on error. */
int hsvd_cu_profile(hsvd_cu_ctx* ctx, int enable);
int64_t hsvd_cu_profile_report(hsvd_cu_ctx* ctx, char* buf, int64_t len);

/* hsvd::validate (svd_factor.cpp:10-21). */
int hsvd_cu_validate(const hsvd_cu_config* cfg);

/* x: m x n row-major with leading dimension ldx, dtype HSVD_CU_F32/F64, in
 * host (where = HSVD_CU_HOST) or device memory.  Result: (sigma, V), u absent.
 *
 * Stream contract for device inputs (where = HSVD_CU_DEVICE, every entry
 * point): the library reads device buffers on the context's stream
 * (hsvd_cu_ctx_stream, created cudaStreamNonBlocking) and does not order
 * itself after any other stream.  The buffer must live on the context's
 * device and be ready on the context's stream when the call is made: a
 * producer on another stream records an event that the context stream waits
 * on (cudaStreamWaitEvent), or synchronizes.  The Python mirror does this for
 * torch tensors (torch's current stream) and rejects tensors on another
 * device.  Host inputs are read synchronously inside the call. */
int hsvd_cu_hierarchical_svd(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                             int64_t ldx, int where, const hsvd_cu_config* cfg,
                             hsvd_cu_result** out);

/* v_r: n x r row-major (ldv), host or device.  Result: (U, sigma, V). */
int hsvd_cu_recover_left_vectors(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                                 int64_t ldx, int where, const double* v_r, int64_t r,
                                 int64_t ldv, int v_where, hsvd_cu_result** out);

/* hsvd::refine_factors (refine.hpp:18-21, refine.cpp:26-72; Alg. 2): v_hat
 * (v_rows x r row-major, v_rows must equal n), sigma_hat (sigma_len = r, host).
 * Result: (U, sigma, V); iterations, final_error (last relative sigma change)
 * and converged as out parameters (non-convergence is not an error). */
int hsvd_cu_refine_factors(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                           int64_t ldx, int where, const double* v_hat, int64_t v_rows,
                           int64_t r, int64_t ldv, int v_where, const double* sigma_hat,
                           int64_t sigma_len, double epsilon, int32_t max_iters,
                           int32_t* iterations, double* final_error, int32_t* converged,
                           hsvd_cu_result** out);

/* ---- device evaluation of reconstruction errors -- */
/* A factor with both sides: u (m x rank), sigma (rank), v (n x rank); host
 * row-major (where = HSVD_CU_HOST, lds in elements) or device column-major
 * (where = HSVD_CU_DEVICE, as returned by hsvd_cu_result_device). */
typedef struct {
  const double* u;
  int64_t ldu;
  const double* sigma;
  const double* v;
  int64_t ldv;
  int64_t m, n, rank;
  int32_t where;
} hsvd_cu_factor_uv;

/* bench.cpp:30-42 factor_diff_norm: ||U_a S_a V_a^T - U_b S_b V_b^T||_F,
 * fused tiles, the m x n difference never stored. */
int hsvd_cu_factor_diff_norm(hsvd_cu_ctx* ctx, const hsvd_cu_factor_uv* a,
                             const hsvd_cu_factor_uv* b, double* out);
/* svd_factor.hpp:61 / svd_factor.cpp:66-80 rank_k_error(full_of_x, approx, k):
 * ||X_k - Xhat_k||_F / ||X_k||_F (same argument checks as the reference). */
int hsvd_cu_rank_k_error(hsvd_cu_ctx* ctx, const hsvd_cu_factor_uv* full_of_x,
                         const hsvd_cu_factor_uv* approx, int64_t k, double* out);
/* ||X - U S V^T||_F for x (m x n row-major, fp32/fp64, host or device). */
int hsvd_cu_residual_norm(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                          int64_t ldx, int where, const hsvd_cu_factor_uv* f, double* out);

/* ---- HSVD1 input streamed to the device --------- */
/* load_hsvd1 (matrix_io.cpp:14-15, 91-113): 22-byte header ("HSVD1\0", u64
 * little-endian rows, u64 cols) and an fp64 row-major payload, streamed in
 * chunks through pinned double buffers straight into device memory owned by
 * the context (kept until the next load or the context's destruction, so it
 * can be passed with HSVD_CU_DEVICE to the calls above).  Same checks and
 * messages as the reference: EIO "cannot open", EFORMAT truncated header /
 * bad magic / empty / implausible dimensions / truncated payload / NaN or
 * Inf (the finiteness check runs on the device). */
int hsvd_cu_load_hsvd1(hsvd_cu_ctx* ctx, const char* path, int64_t* rows, int64_t* cols,
                       const double** dev_x);
/* The same loader also accepting the fp32 payload variant:
 * magic "HSVF1\0", same header, 4-byte little-endian floats (half the file
 * and device bytes of the fp64 form; config 5 is 17 GB instead of 34 GB).
 * *dtype receives HSVD_CU_F32 or HSVD_CU_F64; pass it on with dev_x. */
int hsvd_cu_load_matrix(hsvd_cu_ctx* ctx, const char* path, int64_t* rows, int64_t* cols,
                        int* dtype, const void** dev_x);

/* hierarchical_svd + recover_left_vectors with V_r kept on the device. */
int hsvd_cu_rank_k_svd(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                       int64_t ldx, int where, const hsvd_cu_config* cfg, hsvd_cu_result** out);

int hsvd_cu_svd_of_col_slices(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                              int64_t ldx, int where, int64_t c, double gamma, int64_t max_rank,
                              hsvd_cu_result** out);

/* Result: (U, sigma, V) with p = min(rows, cols) (host row-major input). */
int hsvd_cu_full_svd(hsvd_cu_ctx* ctx, const double* a, int64_t rows, int64_t cols, int64_t lda,
                     hsvd_cu_result** out);

/* orient: HSVD_CU_COLUMN_CONCAT (bases are U) or HSVD_CU_ROW_CONCAT (V). */
int hsvd_cu_merge_pair(hsvd_cu_ctx* ctx, int orient, const hsvd_cu_factor_in* f1,
                       const hsvd_cu_factor_in* f2, double gamma, int64_t max_rank,
                       hsvd_cu_result** out);

int hsvd_cu_tree_merge(hsvd_cu_ctx* ctx, int orient, const hsvd_cu_factor_in* factors,
                       int64_t count, double gamma, int64_t max_rank, int64_t* pair_merges,
                       hsvd_cu_result** out);

/* Building block: top-kk eigenpairs of a symmetric n x n matrix (host,
 * column-major), the device eigensolver every SVD of the path runs on.
 * lam (kk, descending), z (n x kk, column-major). */
int hsvd_cu_syevx_topk(hsvd_cu_ctx* ctx, const double* a, int64_t n, int64_t kk, double* lam,
                       double* z);
/* The same for a batch of `count` matrices in one launch set (the form the
 * leaf stage runs): a = count consecutive n x n matrices, lam = count x kk,
 * z = count consecutive n x kk column-major blocks. */
int hsvd_cu_syevx_topk_batch(hsvd_cu_ctx* ctx, const double* a, int64_t count, int64_t n,
                             int64_t kk, double* lam, double* z);

/* hsvd::qr_thin (kernels.hpp:29, kernels.cpp:50-61): Householder thin QR of
 * the m x n row-major a (host, lda): q (m x p row-major), r (p x n row-major,
 * upper trapezoidal), p = min(m, n); dgeqrf/Eigen sign convention (R_jj =
 * -sign(a_jj) * ||column||).  EINVAL "qr_thin: matrix is empty" for m or n = 0
 * (kernels.cpp:51-53). */
int hsvd_cu_qr_thin(hsvd_cu_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                    double* q, double* r);

/* Building block: the leaf Gram G = X_b^T X_b (c x c, written row-major =
 * column-major, symmetric full storage) of a d x c row-major block, computed
 * as the leaf stage does: fp32 blocks on the tcgen05 int8 tensor cores
 * (Ozaki slices, fp64-grade), fp64 blocks on the fp64 DMMA SYRK. */
int hsvd_cu_block_gram(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t d, int64_t c,
                       int64_t ldx, int where, double* g);

/* ---- multi-GPU (one process / thread per GPU, rows sharded) ---------- */
typedef struct hsvd_cu_group hsvd_cu_group;
/* NCCL: rank 0 creates the 128-byte id and shares it; every rank inits. */
int hsvd_cu_nccl_unique_id(void* out128);
int hsvd_cu_ctx_init_nccl(hsvd_cu_ctx* ctx, int rank, int world, const void* id128);
/* In-process group of contexts driven from separate host threads. */
int hsvd_cu_thread_group_create(int world, hsvd_cu_group** out);
void hsvd_cu_thread_group_free(hsvd_cu_group* g);
int hsvd_cu_ctx_join_group(hsvd_cu_ctx* ctx, hsvd_cu_group* g, int rank);
/* Rows [row0, row0 + m_local) that `rank` must hold: its contiguous row
 * slices of partition(m_total, d) (hierarchy.cpp:11-18). */
int hsvd_cu_shard_rows(int64_t m_total, int64_t d, int rank, int world, int64_t* row0,
                       int64_t* m_local);
/* rank_k_svd over row shards.  Result: U (this rank's m_local rows), sigma
 * and V (replicated on every rank). */
int hsvd_cu_rank_k_svd_sharded(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m_local,
                               int64_t n, int64_t ldx, int where, int64_t m_total, int64_t row0,
                               const hsvd_cu_config* cfg, hsvd_cu_result** out);

/* Result accessors. */
int hsvd_cu_result_info(const hsvd_cu_result* res, int64_t* rank, int32_t* has_u, int32_t* has_v,
                        int64_t* u_rows, int64_t* v_rows, int32_t* degenerate);
int hsvd_cu_result_sigma(const hsvd_cu_result* res, double* out);
int hsvd_cu_result_u(const hsvd_cu_result* res, double* out); /* u_rows x rank, row-major */
int hsvd_cu_result_v(const hsvd_cu_result* res, double* out); /* v_rows x rank, row-major */
int hsvd_cu_result_device(const hsvd_cu_result* res, const double** sigma, const double** u,
                          int64_t* ldu, const double** v, int64_t* ldv); /* column-major */
void hsvd_cu_result_free(hsvd_cu_result* res);

#ifdef __cplusplus
}
#endif

#endif /* HSVD_CU_H_ */
