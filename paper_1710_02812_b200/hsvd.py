"""Python mirror of the reference ``hsvd::core`` API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference library
(``/root/reference/proj/core/include/hsvd``): ``std::invalid_argument`` maps
to ``ValueError`` and ``hsvd::DecompositionError`` to :class:`DecompositionError`.
Every decomposition runs on the GPU through ``libhsvd_b200.so``
(``include/hsvd_cu.h``); there is no CPU fallback -- without the library or a
CUDA device the compute functions raise.

Host-side helpers that the reference implements as plain control logic
(``validate``, ``retained_count``, ``truncate_factor``, ``BlockPlan``,
``reconstruct``, ``normalize_signs``) are restated here directly.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhsvd_b200.so")

OK, EINVAL, EDECOMP, ECUDA, ENCCL, ENOMEM, EIO, EFORMAT = range(8)
F32, F64 = 0, 1
HOST, DEVICE = 0, 1
COLUMN_CONCAT = "ColumnConcat"
ROW_CONCAT = "RowConcat"
_ORIENT = {COLUMN_CONCAT: 0, ROW_CONCAT: 1}


class DecompositionError(RuntimeError):
    """hsvd::DecompositionError (kernels.hpp:12-17)."""

    def __init__(self, what: str, rows: int = 0, cols: int = 0):
        super().__init__(what)
        self.rows = rows
        self.cols = cols


class HsvdCudaError(RuntimeError):
    """CUDA / NCCL / allocation failure inside the library."""


class IoError(RuntimeError):
    """hsvd::IoError (matrix_io.hpp): a matrix file cannot be opened."""


class FormatError(RuntimeError):
    """hsvd::FormatError (matrix_io.hpp): malformed matrix file."""


class _Config(C.Structure):
    _fields_ = [("gamma", C.c_double), ("row_block_rows", C.c_int64),
                ("col_block_cols", C.c_int64), ("epsilon", C.c_double),
                ("max_iters", C.c_int32), ("max_rank", C.c_int64)]


class _FactorIn(C.Structure):
    _fields_ = [("basis", C.POINTER(C.c_double)), ("dim", C.c_int64), ("rank", C.c_int64),
                ("ld", C.c_int64), ("sigma", C.POINTER(C.c_double)),
                ("degenerate", C.c_int32)]


class _FactorUV(C.Structure):
    _fields_ = [("u", C.c_void_p), ("ldu", C.c_int64), ("sigma", C.c_void_p),
                ("v", C.c_void_p), ("ldv", C.c_int64), ("m", C.c_int64), ("n", C.c_int64),
                ("rank", C.c_int64), ("where", C.c_int32)]


_lib = None
_lib_lock = threading.Lock()

# Every symbol include/hsvd_cu.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "hsvd_cu_version", "hsvd_cu_last_error", "hsvd_cu_last_error_dims",
    "hsvd_cu_ctx_create", "hsvd_cu_ctx_destroy", "hsvd_cu_ctx_stream",
    "hsvd_cu_launch_count", "hsvd_cu_arena_bytes", "hsvd_cu_synchronize",
    "hsvd_cu_profile", "hsvd_cu_profile_report",
    "hsvd_cu_validate", "hsvd_cu_hierarchical_svd", "hsvd_cu_recover_left_vectors",
    "hsvd_cu_rank_k_svd", "hsvd_cu_svd_of_col_slices", "hsvd_cu_full_svd",
    "hsvd_cu_merge_pair", "hsvd_cu_tree_merge", "hsvd_cu_result_info",
    "hsvd_cu_result_sigma", "hsvd_cu_result_u", "hsvd_cu_result_v",
    "hsvd_cu_result_device", "hsvd_cu_result_free",
    "hsvd_cu_nccl_unique_id", "hsvd_cu_ctx_init_nccl", "hsvd_cu_thread_group_create",
    "hsvd_cu_thread_group_free", "hsvd_cu_ctx_join_group", "hsvd_cu_shard_rows",
    "hsvd_cu_rank_k_svd_sharded", "hsvd_cu_syevx_topk", "hsvd_cu_refine_factors",
    "hsvd_cu_factor_diff_norm", "hsvd_cu_rank_k_error", "hsvd_cu_residual_norm",
    "hsvd_cu_load_hsvd1", "hsvd_cu_syevx_topk_batch", "hsvd_cu_block_gram",
    "hsvd_cu_qr_thin", "hsvd_cu_load_matrix",
]


def _prefer_bundled_nccl():
    """Points HSVD_NCCL_LIB at the NCCL wheel torch is linked against (the
    library dlopens NCCL lazily; loading an older system libnccl.so.2 first
    would claim the soname and break a later `import torch`)."""
    if os.environ.get("HSVD_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(base, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["HSVD_NCCL_LIB"] = cand
                return
    except Exception:  # pragma: no cover -- optional
        pass


def load_library(path: str = LIB_PATH):
    """Loads libhsvd_b200.so (raises if it has not been built)."""
    _prefer_bundled_nccl()
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `make -C paper_1710_02812_b200` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = C.CDLL(path)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
        pp = C.POINTER(C.c_void_p)
        lib.hsvd_cu_version.restype = I32
        lib.hsvd_cu_last_error.restype = C.c_char_p
        lib.hsvd_cu_last_error_dims.argtypes = [C.POINTER(I64), C.POINTER(I64)]
        lib.hsvd_cu_ctx_create.argtypes = [I32, pp]
        lib.hsvd_cu_ctx_destroy.argtypes = [P]
        lib.hsvd_cu_ctx_stream.argtypes = [P, pp]
        lib.hsvd_cu_launch_count.argtypes = [P]
        lib.hsvd_cu_launch_count.restype = I64
        lib.hsvd_cu_arena_bytes.argtypes = [P]
        lib.hsvd_cu_arena_bytes.restype = I64
        lib.hsvd_cu_synchronize.argtypes = [P]
        lib.hsvd_cu_profile.argtypes = [P, I32]
        lib.hsvd_cu_profile_report.argtypes = [P, C.c_char_p, I64]
        lib.hsvd_cu_profile_report.restype = I64
        lib.hsvd_cu_validate.argtypes = [C.POINTER(_Config)]
        xargs = [P, P, I32, I64, I64, I64, I32]
        lib.hsvd_cu_hierarchical_svd.argtypes = xargs + [C.POINTER(_Config), pp]
        lib.hsvd_cu_rank_k_svd.argtypes = xargs + [C.POINTER(_Config), pp]
        lib.hsvd_cu_recover_left_vectors.argtypes = xargs + [P, I64, I64, I32, pp]
        lib.hsvd_cu_load_hsvd1.argtypes = [P, C.c_char_p, C.POINTER(I64), C.POINTER(I64), pp]
        lib.hsvd_cu_load_matrix.argtypes = [P, C.c_char_p, C.POINTER(I64), C.POINTER(I64),
                                            C.POINTER(C.c_int), pp]
        uv = C.POINTER(_FactorUV)
        lib.hsvd_cu_factor_diff_norm.argtypes = [P, uv, uv, C.POINTER(D)]
        lib.hsvd_cu_rank_k_error.argtypes = [P, uv, uv, I64, C.POINTER(D)]
        lib.hsvd_cu_residual_norm.argtypes = xargs + [uv, C.POINTER(D)]
        lib.hsvd_cu_refine_factors.argtypes = xargs + [P, I64, I64, I64, I32, P, I64, D, I32,
                                                       C.POINTER(I32), C.POINTER(D),
                                                       C.POINTER(I32), pp]
        lib.hsvd_cu_svd_of_col_slices.argtypes = xargs + [I64, D, I64, pp]
        lib.hsvd_cu_full_svd.argtypes = [P, P, I64, I64, I64, pp]
        lib.hsvd_cu_merge_pair.argtypes = [P, I32, C.POINTER(_FactorIn), C.POINTER(_FactorIn),
                                           D, I64, pp]
        lib.hsvd_cu_tree_merge.argtypes = [P, I32, C.POINTER(_FactorIn), I64, D, I64,
                                           C.POINTER(I64), pp]
        lib.hsvd_cu_result_info.argtypes = [P, C.POINTER(I64), C.POINTER(C.c_int32),
                                            C.POINTER(C.c_int32), C.POINTER(I64),
                                            C.POINTER(I64), C.POINTER(C.c_int32)]
        lib.hsvd_cu_result_sigma.argtypes = [P, P]
        lib.hsvd_cu_result_u.argtypes = [P, P]
        lib.hsvd_cu_result_v.argtypes = [P, P]
        lib.hsvd_cu_result_device.argtypes = [P, pp, pp, C.POINTER(I64), pp, C.POINTER(I64)]
        lib.hsvd_cu_result_free.argtypes = [P]
        lib.hsvd_cu_result_free.restype = None
        lib.hsvd_cu_nccl_unique_id.argtypes = [P]
        lib.hsvd_cu_ctx_init_nccl.argtypes = [P, I32, I32, P]
        lib.hsvd_cu_thread_group_create.argtypes = [I32, pp]
        lib.hsvd_cu_thread_group_free.argtypes = [P]
        lib.hsvd_cu_thread_group_free.restype = None
        lib.hsvd_cu_ctx_join_group.argtypes = [P, P, I32]
        lib.hsvd_cu_shard_rows.argtypes = [I64, I64, I32, I32, C.POINTER(I64), C.POINTER(I64)]
        lib.hsvd_cu_rank_k_svd_sharded.argtypes = xargs + [I64, I64, C.POINTER(_Config), pp]
        lib.hsvd_cu_syevx_topk.argtypes = [P, P, I64, I64, P, P]
        lib.hsvd_cu_syevx_topk_batch.argtypes = [P, P, I64, I64, I64, P, P]
        lib.hsvd_cu_block_gram.argtypes = [P, P, I32, I64, I64, I64, I32, P]
        lib.hsvd_cu_qr_thin.argtypes = [P, P, I64, I64, I64, P, P]
        _lib = lib
        return lib


def _raise(code: int):
    lib = load_library()
    msg = lib.hsvd_cu_last_error().decode(errors="replace")
    if code == EINVAL:
        raise ValueError(msg)
    if code == EDECOMP:
        r, c = C.c_int64(), C.c_int64()
        lib.hsvd_cu_last_error_dims(C.byref(r), C.byref(c))
        raise DecompositionError(msg, r.value, c.value)
    if code == EIO:
        raise IoError(msg)
    if code == EFORMAT:
        raise FormatError(msg)
    raise HsvdCudaError(f"[{code}] {msg}")


def _check(code: int):
    if code != OK:
        _raise(code)


# --------------------------------------------------------------------------
# value types (svd_factor.hpp)
# --------------------------------------------------------------------------

@dataclass
class SvdFactor:
    """hsvd::SvdFactor (svd_factor.hpp:14-25)."""

    u: Optional[np.ndarray] = None
    sigma: np.ndarray = field(default_factory=lambda: np.zeros(0))
    v: Optional[np.ndarray] = None
    degenerate: bool = False

    def rank(self) -> int:
        return int(np.asarray(self.sigma).shape[0])

    def has_u(self) -> bool:
        return self.u is not None

    def has_v(self) -> bool:
        return self.v is not None


@dataclass
class MatConfig:
    """hsvd::MatConfig (svd_factor.hpp:28-35)."""

    gamma: float = 1e-2
    row_block_rows: int = 0
    col_block_cols: int = 0
    epsilon: float = 1e-3
    max_iters: int = 10
    max_rank: Optional[int] = None

    def _c(self) -> _Config:
        return _Config(float(self.gamma), int(self.row_block_rows), int(self.col_block_cols),
                       float(self.epsilon), int(self.max_iters),
                       int(self.max_rank) if self.max_rank is not None else 0)


def validate(cfg: MatConfig) -> None:
    """svd_factor.cpp:10-21."""
    if cfg.gamma < 0.0 or not math.isfinite(cfg.gamma):
        raise ValueError("MatConfig: gamma must be finite and >= 0")
    if not (cfg.epsilon > 0.0):
        raise ValueError("MatConfig: epsilon must be > 0")
    if cfg.max_iters < 1:
        raise ValueError("MatConfig: max_iters must be >= 1")
    if cfg.row_block_rows < 0 or cfg.col_block_cols < 0:
        raise ValueError("MatConfig: block sizes must be >= 0")
    if cfg.max_rank is not None and cfg.max_rank < 1:
        raise ValueError("MatConfig: max_rank must be >= 1")


def retained_count(sigma, gamma: float) -> int:
    """svd_factor.cpp:23-30."""
    sigma = np.asarray(sigma)
    if sigma.shape[0] == 0:
        return 0
    if sigma[0] == 0.0:
        return 1
    cutoff = gamma * sigma[0]
    kept = int(np.argmin(sigma >= cutoff)) if not np.all(sigma >= cutoff) else sigma.shape[0]
    return max(kept, 1)


def truncate_factor(f: SvdFactor, gamma: float, max_rank: Optional[int] = None) -> SvdFactor:
    """svd_factor.cpp:32-46."""
    if np.asarray(f.sigma).shape[0] == 0:
        raise ValueError("truncate_factor: factor has an empty spectrum")
    keep = retained_count(f.sigma, gamma)
    if max_rank is not None:
        keep = min(keep, max(int(max_rank), 1))
    return SvdFactor(u=None if f.u is None else f.u[:, :keep].copy(),
                     sigma=np.asarray(f.sigma)[:keep].copy(),
                     v=None if f.v is None else f.v[:, :keep].copy(),
                     degenerate=bool(f.degenerate or f.sigma[0] == 0.0))


def reconstruct(f: SvdFactor) -> np.ndarray:
    """svd_factor.cpp:48-52 (host utility)."""
    if f.u is None or f.v is None:
        raise ValueError("reconstruct: factor must carry both u and v")
    return (f.u * f.sigma) @ f.v.T


def normalize_signs(f: SvdFactor) -> None:
    """svd_factor.cpp:87-104 (host utility)."""
    for j in range(f.rank()):
        side = f.u if f.u is not None else f.v
        if side is None:
            return
        imax = int(np.argmax(np.abs(side[:, j])))
        if side[imax, j] < 0.0:
            if f.u is not None:
                f.u[:, j] = -f.u[:, j]
            if f.v is not None:
                f.v[:, j] = -f.v[:, j]


def partition(extent: int, block: int):
    """hierarchy.cpp:11-18."""
    if block < 1 or block > extent:
        block = extent
    return [(s, min(block, extent - s)) for s in range(0, extent, block)]


@dataclass
class BlockPlan:
    """hsvd::BlockPlan (hierarchy.hpp:18-23)."""

    row_slices: list = field(default_factory=list)
    col_slices: list = field(default_factory=list)

    @staticmethod
    def make(rows: int, cols: int, d: int, c: int) -> "BlockPlan":
        if rows < 1 or cols < 1:
            raise ValueError("BlockPlan: matrix must be nonempty")
        return BlockPlan(partition(rows, d), partition(cols, c))


@dataclass
class MergeStats:
    """hsvd::MergeStats (hierarchy.hpp:25-27)."""

    pair_merges: int = 0


# --------------------------------------------------------------------------
# device context
# --------------------------------------------------------------------------

class Context:
    """One CUDA device + stream + device arena (hsvd_cu_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.hsvd_cu_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if getattr(self, "handle", None):
            self.lib.hsvd_cu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(self.lib.hsvd_cu_ctx_stream(self.handle, C.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        return int(self.lib.hsvd_cu_launch_count(self.handle))

    def arena_bytes(self) -> int:
        return int(self.lib.hsvd_cu_arena_bytes(self.handle))

    def synchronize(self):
        _check(self.lib.hsvd_cu_synchronize(self.handle))

    def profile(self, enable: bool = True):
        """Per-launch CUDA-event timing of the library's kernels."""
        _check(self.lib.hsvd_cu_profile(self.handle, 1 if enable else 0))

    def profile_report(self) -> dict:
        """{'phase[/sub]:kernel': (launches, total_ms, algorithmic_flops)} since
        the last report (flops counted for the GEMM launches, else 0).  The
        algorithmic HBM bytes the library counts for the factor-streaming
        kernels (norms, scale/gather, digit-plane splits) are kept in
        `self.profile_bytes` under the same keys."""
        need = self.lib.hsvd_cu_profile_report(self.handle, None, 0)
        if need < 0:
            _raise(ECUDA)
        buf = C.create_string_buffer(int(need) + 16)
        self.lib.hsvd_cu_profile_report(self.handle, buf, len(buf))
        out = {}
        self.profile_bytes = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms, fl, by = line.split("\t")
            out[name] = (int(cnt), float(ms), float(fl))
            self.profile_bytes[name] = float(by)
        return out


    # --- multi-GPU ---------------------------------------------------------
    def init_nccl(self, rank: int, world: int, unique_id: bytes):
        """Joins an NCCL communicator (one rank per GPU)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(self.lib.hsvd_cu_ctx_init_nccl(self.handle, int(rank), int(world), buf))

    def join_group(self, group: "ThreadGroup", rank: int):
        """Joins an in-process thread group (several contexts, host threads)."""
        _check(self.lib.hsvd_cu_ctx_join_group(self.handle, group.handle, int(rank)))


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    _check(lib.hsvd_cu_nccl_unique_id(buf))
    return buf.raw


class ThreadGroup:
    """In-process communicator group (hsvd_cu_group): lets several host
    threads, each with its own Context, run the sharded pipeline together."""

    def __init__(self, world: int):
        self.lib = load_library()
        h = C.c_void_p()
        _check(self.lib.hsvd_cu_thread_group_create(int(world), C.byref(h)))
        self.handle = h
        self.world = world

    def __del__(self):  # pragma: no cover
        try:
            if self.handle:
                self.lib.hsvd_cu_thread_group_free(self.handle)
        except Exception:
            pass


def shard_rows(m_total: int, d: int, rank: int, world: int):
    """(row0, m_local): the contiguous row slices rank `rank` must hold."""
    lib = load_library()
    r0, ml = C.c_int64(), C.c_int64()
    _check(lib.hsvd_cu_shard_rows(int(m_total), int(d), int(rank), int(world), C.byref(r0),
                                  C.byref(ml)))
    return int(r0.value), int(ml.value)


def rank_k_svd_sharded(x_local, m_total: int, row0: int, cfg: MatConfig, ctx: Context,
                       want_u: bool = True, fetch: bool = True):
    """Sharded rank-k HSVD: this rank holds rows [row0, row0 + len(x_local)).
    Returns SvdFactor with u = this rank's rows of U (or the rank if not fetch)."""
    validate(cfg)
    if x_local is None or (hasattr(x_local, "shape") and x_local.shape[0] == 0):
        n = x_local.shape[1] if x_local is not None else 0
        p, dt, m, ld, where, _keep = None, F64, 0, n, HOST, None
        if x_local is not None and type(x_local).__module__.startswith("torch"):
            dt = F32 if str(x_local.dtype) == "torch.float32" else F64
        elif x_local is not None:
            dt = F32 if np.asarray(x_local).dtype == np.float32 else F64
    else:
        p, dt, m, n, ld, where, _keep = _matrix_arg(x_local, ctx)
    h = C.c_void_p()
    cc = cfg._c()
    _check(ctx.lib.hsvd_cu_rank_k_svd_sharded(ctx.handle, p, dt, m, n, ld, where, int(m_total),
                                              int(row0), C.byref(cc), C.byref(h)))
    if not fetch:
        try:
            rank = C.c_int64()
            _check(ctx.lib.hsvd_cu_result_info(h, C.byref(rank), None, None, None, None, None))
            return int(rank.value)
        finally:
            ctx.lib.hsvd_cu_result_free(h)
    return _result(ctx, h, want_u=want_u)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# --------------------------------------------------------------------------
# marshalling
# --------------------------------------------------------------------------

def _order_after_torch(x, ctx: "Context") -> None:
    """A CUDA tensor is produced on torch's current stream of its device; the
    library reads it on the context's own (non-blocking) stream.  Reject a
    tensor on another device, then make the context stream wait for
    everything already queued on torch's stream (the producer of x, and of
    the .contiguous() copy made here) -- the stream contract of
    HSVD_CU_DEVICE inputs (include/hsvd_cu.h)."""
    import torch
    if x.device.index != ctx.device:
        raise ValueError(f"matrix is on cuda:{x.device.index} but the context is on "
                         f"cuda:{ctx.device}")
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(x.device))
    torch.cuda.ExternalStream(ctx.stream, device=x.device).wait_event(ev)


def _matrix_arg(x, ctx: Optional["Context"] = None):
    """(pointer, dtype code, m, n, ld, where, keepalive) for numpy / torch /
    a DeviceMatrix from load_hsvd1.  CUDA tensors are ordered after torch's
    current stream on the context's stream (ctx defaults to the default
    context)."""
    if isinstance(x, DeviceMatrix):
        return (x.ptr, x.dtype, x.shape[0], x.shape[1], x.shape[1], DEVICE, x)
    mod = type(x).__module__
    if mod.startswith("torch"):
        if x.dim() != 2:
            raise ValueError("matrix must be 2-D")
        if x.stride(1) != 1:
            x = x.contiguous()
        import torch
        dt = {torch.float32: F32, torch.float64: F64}.get(x.dtype)
        if dt is None:
            raise ValueError("matrix dtype must be float32 or float64")
        where = DEVICE if x.is_cuda else HOST
        if x.is_cuda:
            _order_after_torch(x, _ctx(ctx))
        return (x.data_ptr(), dt, x.shape[0], x.shape[1], x.stride(0), where, x)
    a = np.asarray(x)
    if a.ndim != 2:
        raise ValueError("matrix must be 2-D")
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    if not a.flags.c_contiguous or a.strides[1] != a.itemsize:
        a = np.ascontiguousarray(a)
    dt = F32 if a.dtype == np.float32 else F64
    return (a.ctypes.data, dt, a.shape[0], a.shape[1], a.strides[0] // a.itemsize, HOST, a)


def _factor_in(f: SvdFactor, orient: str, keep: list) -> _FactorIn:
    b = f.u if orient == COLUMN_CONCAT else f.v
    if b is None:
        raise ValueError(
            "merge: ColumnConcat requires both factors to carry u" if orient == COLUMN_CONCAT
            else "merge: RowConcat requires both factors to carry v")
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(f.sigma, dtype=np.float64))
    if b.ndim != 2 or b.shape[1] != s.shape[0] or s.shape[0] < 1:
        raise ValueError("merge: basis / sigma shape mismatch")
    keep += [b, s]
    return _FactorIn(b.ctypes.data_as(C.POINTER(C.c_double)), b.shape[0], b.shape[1],
                     b.shape[1], s.ctypes.data_as(C.POINTER(C.c_double)),
                     1 if f.degenerate else 0)


def _result(ctx: Context, h: C.c_void_p, want_u=True, want_v=True) -> SvdFactor:
    lib = ctx.lib
    try:
        rank, hu, hv = C.c_int64(), C.c_int32(), C.c_int32()
        ur, vr, deg = C.c_int64(), C.c_int64(), C.c_int32()
        _check(lib.hsvd_cu_result_info(h, C.byref(rank), C.byref(hu), C.byref(hv),
                                       C.byref(ur), C.byref(vr), C.byref(deg)))
        k = rank.value
        sigma = np.empty(k)
        _check(lib.hsvd_cu_result_sigma(h, sigma.ctypes.data))
        u = v = None
        if hu.value and want_u:
            u = np.empty((ur.value, k))
            _check(lib.hsvd_cu_result_u(h, u.ctypes.data))
        if hv.value and want_v:
            v = np.empty((vr.value, k))
            _check(lib.hsvd_cu_result_v(h, v.ctypes.data))
        return SvdFactor(u=u, sigma=sigma, v=v, degenerate=bool(deg.value))
    finally:
        lib.hsvd_cu_result_free(h)


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# --------------------------------------------------------------------------
# the drop-in API (hierarchy.hpp, merge.hpp, kernels.hpp)
# --------------------------------------------------------------------------

def hierarchical_svd(x, cfg: MatConfig, ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::hierarchical_svd (hierarchy.cpp:65-94) -> (Sigma, V), u absent."""
    validate(cfg)
    c = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, c)
    if m == 0 or n == 0:
        raise ValueError("hierarchical_svd: matrix is empty")
    h = C.c_void_p()
    cc = cfg._c()
    _check(c.lib.hsvd_cu_hierarchical_svd(c.handle, p, dt, m, n, ld, where, C.byref(cc),
                                          C.byref(h)))
    return _result(c, h)


def recover_left_vectors(x, v_r, ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::recover_left_vectors (hierarchy.cpp:96-112) -> (U, Sigma, V)."""
    c = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, c)
    vr = np.ascontiguousarray(np.asarray(v_r, dtype=np.float64))
    if vr.ndim != 2 or vr.shape[0] != n:
        raise ValueError("recover_left_vectors: v_r must have x.cols() rows")
    h = C.c_void_p()
    _check(c.lib.hsvd_cu_recover_left_vectors(c.handle, p, dt, m, n, ld, where, vr.ctypes.data,
                                              vr.shape[1], vr.shape[1], HOST, C.byref(h)))
    return _result(c, h)


@dataclass
class RefineResult:
    """hsvd::RefineResult (refine.hpp:9-14)."""
    factor: SvdFactor
    iterations: int = 0
    final_error: float = 0.0
    converged: bool = False


def refine_factors(x, v_hat, sigma_hat, epsilon: float, max_iters: int,
                   ctx: Optional[Context] = None) -> RefineResult:
    """hsvd::refine_factors (refine.cpp:26-72, Alg. 2): alternate thin SVDs of
    X V and U_outer^T X on the device until the relative sigma change is
    <= epsilon or max_iters is reached; non-convergence is reported."""
    c = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, c)
    vh = np.ascontiguousarray(np.asarray(v_hat, dtype=np.float64))
    sh = np.ascontiguousarray(np.asarray(sigma_hat, dtype=np.float64).reshape(-1))
    if vh.ndim != 2:
        raise ValueError("refine_factors: v_hat must have x.cols() rows")
    it, err, conv = C.c_int(0), C.c_double(0.0), C.c_int(0)
    h = C.c_void_p()
    _check(c.lib.hsvd_cu_refine_factors(c.handle, p, dt, m, n, ld, where, vh.ctypes.data,
                                        vh.shape[0], vh.shape[1], vh.shape[1], HOST,
                                        sh.ctypes.data if sh.size else None, sh.shape[0],
                                        float(epsilon), int(max_iters), C.byref(it),
                                        C.byref(err), C.byref(conv), C.byref(h)))
    return RefineResult(factor=_result(c, h), iterations=int(it.value),
                        final_error=float(err.value), converged=bool(conv.value))


# ---- HSVD1 input streamed to the device -------------

class DeviceMatrix:
    """A matrix resident in device memory owned by a context (the last
    load_hsvd1); accepted wherever a matrix is (passed as HSVD_CU_DEVICE)."""

    def __init__(self, ctx: "Context", ptr: int, rows: int, cols: int, dtype: int = None):
        self.ctx, self.ptr, self.shape = ctx, ptr, (rows, cols)
        self.dtype = F64 if dtype is None else dtype


def load_hsvd1(path: str, ctx: Optional[Context] = None) -> DeviceMatrix:
    """matrix_io.cpp:91-113 load_hsvd1, streamed straight to the device (IoError /
    FormatError with the reference's messages)."""
    c = _ctx(ctx)
    r, k = C.c_int64(), C.c_int64()
    ptr = C.c_void_p()
    _check(c.lib.hsvd_cu_load_hsvd1(c.handle, os.fsencode(path), C.byref(r), C.byref(k),
                                    C.byref(ptr)))
    return DeviceMatrix(c, ptr.value, int(r.value), int(k.value))


def load_matrix(path: str, ctx: Optional[Context] = None) -> DeviceMatrix:
    """load_hsvd1 also accepting the fp32 payload variant ("HSVF1\0" magic,
    same header): the matrix stays fp32 on the device."""
    c = _ctx(ctx)
    r, k, dt = C.c_int64(), C.c_int64(), C.c_int(0)
    ptr = C.c_void_p()
    _check(c.lib.hsvd_cu_load_matrix(c.handle, os.fsencode(path), C.byref(r), C.byref(k),
                                     C.byref(dt), C.byref(ptr)))
    return DeviceMatrix(c, ptr.value, int(r.value), int(k.value), int(dt.value))


def save_hsvd1(x, path: str, dtype: str = "f64") -> None:
    """matrix_io.cpp:115-127 save_hsvd1 (host writer, for tests and the CLI);
    dtype="f32" writes the fp32 payload variant (magic "HSVF1\0")."""
    f32 = dtype == "f32"
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32 if f32 else np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    with open(path, "wb") as f:
        f.write((b"HSVF1\0" if f32 else b"HSVD1\0") + int(a.shape[0]).to_bytes(8, "little") +
                int(a.shape[1]).to_bytes(8, "little"))
        f.write(a.astype("<f4" if f32 else "<f8").tobytes())


# ---- device evaluation of reconstruction errors -----

def _uv(f: SvdFactor, who: str):
    """(struct, keep-alive arrays) for a host factor with both sides."""
    if f.u is None or f.v is None:
        raise ValueError(f"{who}: factor must carry both u and v")
    u = np.ascontiguousarray(np.asarray(f.u, dtype=np.float64))
    v = np.ascontiguousarray(np.asarray(f.v, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(f.sigma, dtype=np.float64).reshape(-1))
    st = _FactorUV(u.ctypes.data, u.shape[1], s.ctypes.data, v.ctypes.data, v.shape[1],
                   u.shape[0], v.shape[0], s.shape[0], HOST)
    return st, (u, v, s)


def factor_diff_norm(a: SvdFactor, b: SvdFactor, ctx: Optional[Context] = None) -> float:
    """bench.cpp:30-42: ||U_a S_a V_a^T - U_b S_b V_b^T||_F on the device (fused
    tiles; the m x n difference is never stored)."""
    c = _ctx(ctx)
    sa, ka = _uv(a, "factor_diff_norm")
    sb, kb = _uv(b, "factor_diff_norm")
    out = C.c_double(0.0)
    _check(c.lib.hsvd_cu_factor_diff_norm(c.handle, C.byref(sa), C.byref(sb), C.byref(out)))
    return float(out.value)


def rank_k_error(full_of_x_or_x, approx: SvdFactor, k: int,
                 ctx: Optional[Context] = None) -> float:
    """hsvd::rank_k_error (svd_factor.cpp:66-83): ||X_k - Xhat_k||_F / ||X_k||_F,
    evaluated on the device.  The first argument is the full SVD of X or X
    itself (then decomposed by full_svd first, as the reference does)."""
    c = _ctx(ctx)
    if approx.u is None or approx.v is None:
        raise ValueError("rank_k_error: approx must carry both u and v")
    full = full_of_x_or_x if isinstance(full_of_x_or_x, SvdFactor) else full_svd(full_of_x_or_x, c)
    sf, kf = _uv(full, "rank_k_error")
    sa, ka = _uv(approx, "rank_k_error")
    out = C.c_double(0.0)
    _check(c.lib.hsvd_cu_rank_k_error(c.handle, C.byref(sf), C.byref(sa), int(k), C.byref(out)))
    return float(out.value)


def residual_norm(x, f: SvdFactor, ctx: Optional[Context] = None) -> float:
    """||X - U S V^T||_F on the device (x host/device, fp32/fp64)."""
    c = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, c)
    sf, kf = _uv(f, "residual_norm")
    out = C.c_double(0.0)
    _check(c.lib.hsvd_cu_residual_norm(c.handle, p, dt, m, n, ld, where, C.byref(sf),
                                       C.byref(out)))
    return float(out.value)


def rank_k_svd(x, cfg: MatConfig, ctx: Optional[Context] = None, want_u: bool = True) -> SvdFactor:
    """hierarchical_svd + recover_left_vectors in one device-resident call."""
    validate(cfg)
    c = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, c)
    h = C.c_void_p()
    cc = cfg._c()
    _check(c.lib.hsvd_cu_rank_k_svd(c.handle, p, dt, m, n, ld, where, C.byref(cc), C.byref(h)))
    return _result(c, h, want_u=want_u)


def rank_k_svd_device(x, cfg: MatConfig, ctx: Context) -> int:
    """rank_k_svd with the result left in device memory (benchmarks): returns
    the rank; no host copies are made."""
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, ctx)
    h = C.c_void_p()
    cc = cfg._c()
    _check(ctx.lib.hsvd_cu_rank_k_svd(ctx.handle, p, dt, m, n, ld, where, C.byref(cc),
                                      C.byref(h)))
    try:
        rank = C.c_int64()
        _check(ctx.lib.hsvd_cu_result_info(h, C.byref(rank), None, None, None, None, None))
        return int(rank.value)
    finally:
        ctx.lib.hsvd_cu_result_free(h)


def syevx_topk(a, kk: int, ctx: Optional[Context] = None):
    """Top-kk eigenpairs of a symmetric matrix on the device eigensolver
    (the building block of every SVD in the path): (lam desc, Z n x kk)."""
    cx = _ctx(ctx)
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    lam = np.empty(kk)
    z = np.empty((kk, n))  # column-major n x kk == row-major kk x n
    _check(cx.lib.hsvd_cu_syevx_topk(cx.handle, a.ctypes.data, n, int(kk), lam.ctypes.data,
                                     z.ctypes.data))
    return lam, z.T.copy()


def syevx_topk_batch(a, kk: int, ctx: Optional[Context] = None):
    """Top-kk eigenpairs of a batch of symmetric matrices (count x n x n) in
    one launch set: (lam count x kk desc, Z count x n x kk)."""
    cx = _ctx(ctx)
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    count, n = a.shape[0], a.shape[1]
    lam = np.empty((count, kk))
    z = np.empty((count, kk, n))  # per matrix column-major n x kk
    _check(cx.lib.hsvd_cu_syevx_topk_batch(cx.handle, a.ctypes.data, count, n, int(kk),
                                           lam.ctypes.data, z.ctypes.data))
    return lam, np.ascontiguousarray(z.transpose(0, 2, 1))


def qr_thin(a, ctx: Optional[Context] = None):
    """hsvd::qr_thin (kernels.cpp:50-61): Householder thin QR on the device,
    (q rows x p, r p x cols), p = min(rows, cols)."""
    cx = _ctx(ctx)
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("qr_thin: matrix is empty")
    m, n = a.shape
    p = min(m, n)
    q = np.empty((m, p))
    r = np.empty((p, n))
    _check(cx.lib.hsvd_cu_qr_thin(cx.handle, a.ctypes.data, m, n, n, q.ctypes.data,
                                  r.ctypes.data))
    return q, r


def block_gram(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Leaf Gram X^T X of a d x c block as the leaf stage computes it (fp32:
    tcgen05 int8 Ozaki slices; fp64: DMMA SYRK)."""
    cx = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x, cx)
    g = np.empty((n, n))
    _check(cx.lib.hsvd_cu_block_gram(cx.handle, p, dt, m, n, ld, where, g.ctypes.data))
    return g


def svd_of_col_slices(x_slice, c: int, gamma: float, max_rank: Optional[int] = None,
                      ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::svd_of_col_slices (hierarchy.cpp:50-63) -> (U, Sigma), v absent."""
    cx = _ctx(ctx)
    p, dt, m, n, ld, where, _keep = _matrix_arg(x_slice, cx)
    h = C.c_void_p()
    _check(cx.lib.hsvd_cu_svd_of_col_slices(cx.handle, p, dt, m, n, ld, where, int(c),
                                            float(gamma), int(max_rank or 0), C.byref(h)))
    return _result(cx, h)


def full_svd(a, ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::full_svd (kernels.cpp:21-48): thin SVD, p = min(rows, cols)."""
    cx = _ctx(ctx)
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("full_svd: matrix is empty")
    h = C.c_void_p()
    _check(cx.lib.hsvd_cu_full_svd(cx.handle, a.ctypes.data, a.shape[0], a.shape[1], a.shape[1],
                                   C.byref(h)))
    return _result(cx, h)


def _merge(f1: SvdFactor, f2: SvdFactor, orient: str, gamma: float, max_rank, ctx) -> SvdFactor:
    cx = _ctx(ctx)
    keep: list = []
    a = _factor_in(f1, orient, keep)
    b = _factor_in(f2, orient, keep)
    if a.dim != b.dim:
        raise ValueError("merge: ColumnConcat factors must have equal row counts"
                         if orient == COLUMN_CONCAT else
                         "merge: RowConcat factors must have equal column counts")
    h = C.c_void_p()
    _check(cx.lib.hsvd_cu_merge_pair(cx.handle, _ORIENT[orient], C.byref(a), C.byref(b),
                                     float(gamma), int(max_rank or 0), C.byref(h)))
    return _result(cx, h)


def merge_pair_qr(f1: SvdFactor, f2: SvdFactor, orient: str, gamma: float,
                  max_rank: Optional[int] = None, ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::merge_pair_qr (merge.cpp:71-117); on the GPU both merges compute
    the SVD of [B1 S1 | B2 S2] through its (k+l)^2 Gram."""
    return _merge(f1, f2, orient, gamma, max_rank, ctx)


def merge_pair_naive(f1: SvdFactor, f2: SvdFactor, orient: str, gamma: float,
                     max_rank: Optional[int] = None, ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::merge_pair_naive (merge.cpp:42-69)."""
    return _merge(f1, f2, orient, gamma, max_rank, ctx)


def tree_merge(factors: Sequence[SvdFactor], orient: str, gamma: float,
               max_rank: Optional[int] = None, stats: Optional[MergeStats] = None,
               ctx: Optional[Context] = None) -> SvdFactor:
    """hsvd::tree_merge (hierarchy.cpp:31-48)."""
    factors = list(factors)
    if not factors:
        raise ValueError("tree_merge: factor list is empty")
    if len(factors) == 1:
        return factors[0]
    cx = _ctx(ctx)
    keep: list = []
    arr = (_FactorIn * len(factors))(*[_factor_in(f, orient, keep) for f in factors])
    pm = C.c_int64()
    h = C.c_void_p()
    _check(cx.lib.hsvd_cu_tree_merge(cx.handle, _ORIENT[orient], arr, len(factors), float(gamma),
                                     int(max_rank or 0), C.byref(pm), C.byref(h)))
    if stats is not None:
        stats.pair_merges += int(pm.value)
    return _result(cx, h)
