"""Block-grid benchmark report with GPU timings.

Restates the reference's ``run_benchmark`` / ``report_to_json`` /
``validate_report_json`` (bench.hpp:13-62, bench.cpp:68-270) and the cost
model (cost_model.hpp:22-60) over the device API: the full-SVD baseline,
the hierarchical pipeline, the refined pipeline and the error metric all run
on the B200 (``full_svd``, ``hierarchical_svd`` + ``recover_left_vectors``,
``refine_factors``, ``factor_diff_norm``); the wall times are of those
device calls.  ``kernel_threads`` records the streaming-multiprocessor
count the kernels ran on (the reference records Eigen's thread count).
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import hsvd as _h


# --------------------------------------------------------------------------
# cost model (cost_model.hpp:22-60, paper section 3.1)
# --------------------------------------------------------------------------

@dataclass
class CostEstimate:
    flops_full: float = 0.0
    flops_mat: float = 0.0
    bound: float = 0.0
    partitions: int = 0        # P
    cols_per_block: float = 0.0  # s = n / P
    merge_rank: int = 0        # k


def flops_full_svd(m: int, n: int) -> float:
    """cost_model.hpp:22-27: 6 m n^2 + 16 n^3 (tall orientation)."""
    if m < n or n < 1:
        raise ValueError("flops_full_svd: requires m >= n >= 1 (pass the tall orientation)")
    return 6.0 * m * n * n + 16.0 * float(n) ** 3


def flops_mat_partition(m: int, n: int, p: int, k: int) -> float:
    """cost_model.hpp:31-40: P (6 m s^2 + 16 s^3) + (P-1)(14 m k^2 + 176 k^3)."""
    if p < 1:
        raise ValueError("flops_mat_partition: P must be >= 1")
    s = n / p
    if s < 1.0:
        raise ValueError("flops_mat_partition: requires s = n/P >= 1")
    if k > s:
        raise ValueError("flops_mat_partition: model assumes k <= s")
    return p * (6.0 * m * s * s + 16.0 * s ** 3) + (p - 1.0) * (14.0 * m * k * k + 176.0 * float(k) ** 3)


def speedup_bound(m: int, n: int, p: int) -> float:
    """cost_model.hpp:44-49: 20 m n^2 / P + 192 n^3 / P^2."""
    if p < 1:
        raise ValueError("speedup_bound: P must be >= 1")
    return 20.0 * m * n * n / p + 192.0 * float(n) ** 3 / (p * p)


def estimate_costs(m: int, n: int, p: int, k: int) -> CostEstimate:
    """cost_model.hpp:51-60."""
    return CostEstimate(flops_full=flops_full_svd(max(m, n), min(m, n)),
                        flops_mat=flops_mat_partition(m, n, p, k),
                        bound=speedup_bound(m, n, p), partitions=p, cols_per_block=n / p,
                        merge_rank=k)


# --------------------------------------------------------------------------
# run_benchmark (bench.cpp:68-156)
# --------------------------------------------------------------------------

@dataclass
class GridPoint:
    block_rows: int = 0  # d
    block_cols: int = 0  # c


@dataclass
class BenchEntry:
    block_rows: int = 0
    block_cols: int = 0
    error: str = ""
    recovered_rank: int = 0
    wall_time_mat_s: float = 0.0
    wall_time_full_svd_s: float = 0.0
    speedup: float = 0.0
    rel_error: float = 0.0
    wall_time_mat_refined_s: Optional[float] = None
    speedup_refined: Optional[float] = None
    rel_error_refined: Optional[float] = None
    sigma_head: List[float] = field(default_factory=list)
    predicted: Optional[CostEstimate] = None


@dataclass
class BenchReport:
    rows: int = 0
    cols: int = 0
    gamma: float = 0.0
    epsilon: float = 0.0
    repeats: int = 1
    kernel_threads: int = 1
    entries: List[BenchEntry] = field(default_factory=list)


def _head(f: "_h.SvdFactor", k: int) -> "_h.SvdFactor":
    return _h.SvdFactor(u=f.u[:, :k], sigma=np.asarray(f.sigma)[:k], v=f.v[:, :k])


def rel_error_against(full, approx, k: int, ctx=None) -> float:
    """bench.cpp:52-58: ||X_k - Xhat_k||_F / ||Sigma_k|| with the difference
    evaluated on the device (factor_diff_norm)."""
    k_ref = min(k, full.rank())
    ref = _head(full, k_ref)
    denom = math.sqrt(float(np.sum(np.asarray(ref.sigma) ** 2)))
    if denom == 0.0:
        raise ValueError("rel_error: reference rank-k matrix is zero")
    return _h.factor_diff_norm(ref, _head(approx, min(k, approx.rank())), ctx) / denom


def _device_input(x):
    """The matrix once in HBM (torch), so the timed calls exclude the upload."""
    try:
        import torch
        if torch.cuda.is_available():
            return torch.as_tensor(np.ascontiguousarray(x)).cuda()
    except ImportError:  # pragma: no cover
        pass
    return x


def run_benchmark(x, cfg: "_h.MatConfig", grid: List[GridPoint], repeats: int,
                  with_refine: bool = True, ctx=None) -> BenchReport:
    """bench.cpp:68-156 over the device API (per-entry failures recorded)."""
    if not grid:
        raise ValueError("run_benchmark: grid is empty")
    if repeats < 1:
        raise ValueError("run_benchmark: repeats must be >= 1")
    _h.validate(cfg)
    c = _h._ctx(ctx)
    x = np.asarray(x, dtype=np.float64)
    import torch
    report = BenchReport(rows=x.shape[0], cols=x.shape[1], gamma=cfg.gamma, epsilon=cfg.epsilon,
                         repeats=repeats,
                         kernel_threads=int(torch.cuda.get_device_properties(c.device)
                                            .multi_processor_count))
    xd = _device_input(x)
    base_total = 0.0
    full = None
    for _ in range(repeats):
        t0 = time.perf_counter()
        full = _h.full_svd(x, c)
        base_total += time.perf_counter() - t0
    base_mean = base_total / repeats
    for gp in grid:
        entry = BenchEntry(block_rows=gp.block_rows, block_cols=gp.block_cols)
        try:
            run_cfg = _h.MatConfig(gamma=cfg.gamma, row_block_rows=gp.block_rows,
                                   col_block_cols=gp.block_cols, epsilon=cfg.epsilon,
                                   max_iters=cfg.max_iters, max_rank=cfg.max_rank)
            _h.validate(run_cfg)
            mat_total = refined_total = 0.0
            approx = refined = None
            for _ in range(repeats):
                t0 = time.perf_counter()
                right = _h.hierarchical_svd(xd, run_cfg, c)
                t_hier = time.perf_counter() - t0
                t0 = time.perf_counter()
                approx = _h.recover_left_vectors(xd, right.v, c)
                mat_total += t_hier + time.perf_counter() - t0
                if with_refine:
                    t0 = time.perf_counter()
                    refined = _h.refine_factors(xd, right.v, right.sigma, run_cfg.epsilon,
                                                run_cfg.max_iters, c)
                    refined_total += t_hier + time.perf_counter() - t0
            entry.recovered_rank = approx.rank()
            entry.wall_time_mat_s = mat_total / repeats
            entry.wall_time_full_svd_s = base_mean
            entry.speedup = base_mean / entry.wall_time_mat_s
            entry.rel_error = rel_error_against(full, approx, approx.rank(), c)
            entry.sigma_head = [float(s) for s in np.asarray(approx.sigma)[:64]]
            if with_refine:
                entry.wall_time_mat_refined_s = refined_total / repeats
                entry.speedup_refined = base_mean / entry.wall_time_mat_refined_s
                entry.rel_error_refined = rel_error_against(full, refined.factor,
                                                            approx.rank(), c)
            p = max(1, -(-x.shape[1] // max(gp.block_cols, 1)))
            model_k = min(entry.recovered_rank, x.shape[1] // p)
            entry.predicted = estimate_costs(x.shape[0], x.shape[1], p, max(model_k, 1))
        except Exception as err:  # noqa: BLE001 -- recorded per entry (bench.cpp:146-151)
            entry = BenchEntry(block_rows=gp.block_rows, block_cols=gp.block_cols,
                               error=str(err) or type(err).__name__)
        report.entries.append(entry)
    return report


# --------------------------------------------------------------------------
# JSON report (bench.cpp:158-270, docs/bench_report.schema.json)
# --------------------------------------------------------------------------

def _cost_json(est: CostEstimate) -> dict:
    return {"flops_full": est.flops_full, "flops_mat": est.flops_mat, "bound": est.bound,
            "P": est.partitions, "s": est.cols_per_block, "k": est.merge_rank}


def report_to_json(report: BenchReport, indent: int = 2) -> str:
    """bench.cpp:158-188."""
    entries = []
    for e in report.entries:
        j = {"block_rows": e.block_rows, "block_cols": e.block_cols}
        if e.error:
            j["error"] = e.error
        else:
            j.update({"recovered_rank": e.recovered_rank, "wall_time_mat_s": e.wall_time_mat_s,
                      "wall_time_full_svd_s": e.wall_time_full_svd_s, "speedup": e.speedup,
                      "rel_error": e.rel_error, "sigma_head": list(e.sigma_head)})
            if e.predicted is not None:
                j["predicted"] = _cost_json(e.predicted)
            if e.wall_time_mat_refined_s is not None:
                j["wall_time_mat_refined_s"] = e.wall_time_mat_refined_s
                j["speedup_refined"] = e.speedup_refined
                j["rel_error_refined"] = e.rel_error_refined
        entries.append(j)
    root = {"matrix_dims": [report.rows, report.cols], "gamma": report.gamma,
            "epsilon": report.epsilon, "repeats": report.repeats,
            "kernel_threads": report.kernel_threads, "grid": entries}
    return json.dumps(root, indent=indent) + "\n"


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def validate_report_json(text: str) -> List[str]:
    """bench.cpp:198-270: one message per violation, empty = valid."""
    try:
        root = json.loads(text)
    except (ValueError, TypeError):
        return ["not valid JSON"]
    if not isinstance(root, dict):
        return ["root is not an object"]
    out: List[str] = []

    def req(ok: bool, msg: str):
        if not ok:
            out.append(msg)

    md = root.get("matrix_dims")
    req(isinstance(md, list) and len(md) == 2 and all(_is_int(v) for v in md),
        "matrix_dims must be a [rows, cols] integer pair")
    for key in ("gamma", "epsilon"):
        req(_is_num(root.get(key)), f"{key} must be a number")
    for key in ("repeats", "kernel_threads"):
        req(_is_int(root.get(key)), f"{key} must be an integer")
    grid = root.get("grid")
    if not isinstance(grid, list):
        out.append("grid must be an array")
        return out
    for idx, e in enumerate(grid):
        at = f"grid[{idx}]: "
        if not isinstance(e, dict):
            out.append(at + "entry is not an object")
            continue
        for key in ("block_rows", "block_cols"):
            req(_is_int(e.get(key)), at + f"{key} must be an integer")
        if "error" in e:
            req(isinstance(e["error"], str) and e["error"] != "",
                at + "error must be a nonempty string")
            continue
        req(_is_int(e.get("recovered_rank")), at + "recovered_rank must be an integer")
        for key in ("wall_time_mat_s", "wall_time_full_svd_s", "speedup", "rel_error"):
            req(_is_num(e.get(key)), at + f"{key} must be a number")
        head = e.get("sigma_head")
        head_ok = isinstance(head, list) and len(head) <= 64
        req(head_ok, at + "sigma_head must be an array of <= 64 numbers")
        if head_ok and not all(_is_num(s) for s in head):
            out.append(at + "sigma_head holds a non-number")
        if "predicted" in e:
            p = e["predicted"]
            req(isinstance(p, dict), at + "predicted must be an object")
            if isinstance(p, dict):
                for key in ("flops_full", "flops_mat", "bound", "s"):
                    req(_is_num(p.get(key)), at + f"predicted.{key} must be a number")
                for key in ("P", "k"):
                    req(_is_int(p.get(key)), at + f"predicted.{key} must be an integer")
        keys = ("wall_time_mat_refined_s", "speedup_refined", "rel_error_refined")
        if any(k in e for k in keys):
            for key in keys:
                req(_is_num(e.get(key)),
                    at + f"refined metrics must be present together and numeric ({key})")
    return out


def main(argv=None) -> int:
    """`bench` of the reference CLI (hsvd_main.cpp:161-190, options :268-279):
    python -m paper_1710_02812_b200.report --input X.hsvd --grid d1xc1,... [--json P]."""
    import argparse
    import sys
    ap = argparse.ArgumentParser(prog="python -m paper_1710_02812_b200.report")
    ap.add_argument("--input", required=True)
    ap.add_argument("--gamma", type=float, default=1e-2)
    ap.add_argument("--grid", required=True)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--refine", action="store_true")
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--max-iters", type=int, default=10)
    ap.add_argument("--json", default="")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        grid = []
        for item in a.grid.split(","):
            d, c = item.split("x")
            if int(d) <= 0 or int(c) <= 0:
                raise ValueError
            grid.append(GridPoint(int(d), int(c)))
    except ValueError:
        print(f"--grid: expected d1xc1,d2xc2,... got '{a.grid}'", file=sys.stderr)
        return 1
    try:
        dm = _h.load_hsvd1(a.input)  # the reference's checks (matrix_io.cpp:91-113)
        x = np.fromfile(a.input, dtype="<f8", offset=22).reshape(dm.shape)
        rep = run_benchmark(x, _h.MatConfig(gamma=a.gamma, epsilon=a.eps,
                                            max_iters=a.max_iters), grid, a.repeats, a.refine)
    except Exception as err:  # noqa: BLE001
        print(f"error: {err}", file=sys.stderr)
        return 2
    for e in rep.entries:
        if e.error:
            print(f"{e.block_rows}x{e.block_cols}: error: {e.error}")
        else:
            print(f"{e.block_rows}x{e.block_cols}: rank {e.recovered_rank}, "
                  f"{e.wall_time_mat_s:.6g} s (full SVD {e.wall_time_full_svd_s:.6g} s, "
                  f"speedup {e.speedup:.6g}), rel error {e.rel_error:.6g}")
    if a.json:
        with open(a.json, "w") as f:
            f.write(report_to_json(rep))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
