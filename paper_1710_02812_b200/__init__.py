"""B200-native hierarchical merge-and-truncate SVD (arXiv 1710.02812).

Drop-in for the hot path of the reference ``hsvd::core`` library:
``hierarchical_svd`` followed by ``recover_left_vectors``, computed by
hand-written sm_100a CUDA kernels in ``libhsvd_b200.so`` behind the C ABI in
``include/hsvd_cu.h``.
"""
from .hsvd import (  # noqa: F401
    COLUMN_CONCAT, ROW_CONCAT, BlockPlan, Context, DecompositionError, HsvdCudaError,
    MatConfig, MergeStats, SvdFactor, default_context, full_svd, hierarchical_svd,
    load_library, merge_pair_naive, merge_pair_qr, normalize_signs, partition,
    rank_k_svd, rank_k_svd_device, reconstruct, recover_left_vectors, retained_count, svd_of_col_slices,
    tree_merge, truncate_factor, validate, LIB_PATH, EXPORTED, ThreadGroup, nccl_unique_id,
    shard_rows, rank_k_svd_sharded, syevx_topk, syevx_topk_batch, block_gram, qr_thin, refine_factors, RefineResult,
    factor_diff_norm, rank_k_error, residual_norm, load_hsvd1, load_matrix, save_hsvd1, DeviceMatrix,
    IoError, FormatError,
)
