#!/usr/bin/env python
"""Benchmark of the rank-k HSVD hot path (hierarchical_svd + recover_left_vectors).

Metric (BASELINE.json): HSVD input GB/s = m*n*sizeof(dtype) / t per rank-k
SVD, whole job.  One step = one full rank-k HSVD of the workload matrix.
Default workload: BASELINE config 5 (65536x65536 fp32, 16x16 grid, k=200),
the largest configuration that fits one B200.

  python bench.py [--gpus N --steps K --warmup W --config C]
  python bench.py --impl reference ...   (CPU oracle arm, rank 0 only)

--gpus N without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1).

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
cudaStreamSynchronize, CUDA events on the library's stream, max over ranks.
The input (>= 1.6 GB for configs 2-5) exceeds the 126 MB L2, so no flush is
needed between steps (stated in "config").
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HSVD input GB/s (and time to rank-k SVD), % of roofline"
GAMMA = 1e-12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-single", action="store_true",
                    help="skip the single-thread CPU leaf timing")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="(CPU tests) spawn --gpus ranks over gloo, rendezvous, print n_gpus")
    return ap.parse_args()


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(args) -> int:
    """--gpus N > WORLD_SIZE: run this script under torch.distributed.run with
    N ranks on this node (the same command the driver uses for N > 1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    return subprocess.call(cmd, env=env)


def launcher_selftest(args) -> int:
    """Rank body of --launcher-selftest: gloo rendezvous + an all-reduce, then
    rank 0 prints the contract's n_gpus."""
    import torch
    import torch.distributed as dist
    ws, rank, _ = dist_env()
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "world_size": dist.get_world_size(),
                          "max_rank_plus_1": float(t.item())}), flush=True)
    dist.destroy_process_group()
    return 0


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU arm (oracle port on the host cores)
# ---------------------------------------------------------------------------

def host_leaves(w, count):
    """The first `count` leaf blocks of row slice 0 (host fp32/fp64 copies) of
    the exact matrix the GPU arm times: generated on cuda:0 with the bench's
    generator and seed.  Without a GPU (CPU tests) the numpy generator of the
    same recipe stands in; the returned description says which."""
    from paper_1710_02812_b200 import configs
    count = max(1, min(count, w.Q))
    try:
        import torch
        cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        cuda = False
    if cuda:
        x = configs.generate_torch(w, device=torch.device("cuda", 0))
        blocks = [x[:w.d, j * w.c:(j + 1) * w.c].cpu().numpy() for j in range(count)]
        full = x.cpu().numpy() if w.input_bytes <= (64 << 20) else None
        del x
        torch.cuda.empty_cache()
        src = "bytes of configs.generate_torch on cuda:0 (the GPU arm's input)"
    else:
        full = configs.generate_numpy(w)
        blocks = [full[:w.d, j * w.c:(j + 1) * w.c].copy() for j in range(count)]
        src = "configs.generate_numpy (no GPU on this host)"
    return blocks, full, src


def whole_pipeline_fits(w):
    """Small workloads (config 1) run the complete reference pipeline per step."""
    return w.input_bytes <= (64 << 20)


def cpu_step(w, blocks, full, i, threads):
    """One CPU step of the reference algorithm (oracle port): the complete
    rank-k HSVD (hierarchical_svd + recover_left_vectors, hierarchy.cpp:65-112)
    when the workload is small, else leaf i of row slice 0 through full_svd +
    truncate_factor (hierarchy.cpp:57, kernels.cpp:21-48) -- the leaf SVDs
    are > 95% of the reference's flops at configs 2-5; the
    column/row merges and the recoveries are not in this sample.
    Returns (seconds, bytes of X covered, description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import hsvd_oracle as O
    from threadpoolctl import threadpool_limits
    if full is not None and whole_pipeline_fits(w):
        cfg = O.MatConfig(gamma=GAMMA, row_block_rows=w.d, col_block_cols=w.c, max_rank=w.k)
        t0 = time.perf_counter()
        with threadpool_limits(1):
            r = O.hierarchical_svd(full, cfg, workers=threads)
        with threadpool_limits(threads):
            O.recover_left_vectors(full, r.v)
        sec = time.perf_counter() - t0
        return sec, full.nbytes, (f"complete rank-k HSVD of the {w.m}x{w.n} matrix "
                                  f"(hierarchical_svd + recover_left_vectors), numpy/LAPACK "
                                  f"oracle port, {threads} threads")
    blk = blocks[i % len(blocks)]
    t0 = time.perf_counter()
    with threadpool_limits(threads):
        f = O.full_svd(np.asarray(blk, dtype=np.float64))
        O.truncate_factor(f, GAMMA, w.k)
    sec = time.perf_counter() - t0
    return sec, blk.nbytes, (f"one {w.d}x{w.c} leaf of row slice 0 per step (leaf "
                             f"{i % len(blocks)}), full_svd + truncate_factor, numpy/LAPACK "
                             f"(dgesdd) oracle port, {threads} threads; merges and recoveries "
                             f"(< 5% of the reference's flops) not sampled")


def arm_config(w, ws):
    """The workload description both arms print."""
    return {"workload": w.name, "m": w.m, "n": w.n, "input_dtype": w.dtype,
            "grid": f"{w.P}x{w.Q}", "k": w.k, "gamma": GAMMA,
            "l2": "input exceeds the 126 MB L2; no flush between steps",
            "parallelism": (f"rows sharded by row slice over {ws} GPUs (NCCL)"
                            if ws > 1 else "single GPU")}


def run_reference(args, w):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = args.cpu_threads or os.cpu_count() or 1
    blocks, full, src = host_leaves(w, args.warmup + args.steps)
    times, nbytes = [], []
    desc = ""
    for i in range(args.warmup + args.steps):
        sec, nb, desc = cpu_step(w, blocks, full, i, threads)
        if i >= args.warmup:
            times.append(sec)
            nbytes.append(nb)
    ms = 1000.0 * statistics.mean(times)
    value = sum(nbytes) / sum(times) / 1e9
    desc = f"{desc}; input: {src}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json recipe)",
        "config": dict(arm_config(w, 1), sample=desc,
                       parallelism=f"CPU oracle port, {threads} host threads"),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": desc},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args, w):
    """cpu_baseline of the GPU arm (rank 0, N=1): one sample step on all host
    threads, plus the reference's own single-thread mode (Eigen runs
    single-threaded, bench.cpp:81) on one leaf."""
    threads = args.cpu_threads or os.cpu_count() or 1
    blocks, full, src = host_leaves(w, 1)
    sec, nb, desc = cpu_step(w, blocks, full, 0, threads)
    out = {"value": nb / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
           "sample": f"{desc}; input: {src}", "seconds": sec}
    if not args.no_cpu_single:
        sec1, nb1, desc1 = cpu_step(w, blocks, full, 0, 1)
        out["single_thread"] = {"value": nb1 / sec1 / 1e9, "unit": "GB/s", "cores": 1,
                                "seconds": sec1, "sample": desc1}
    return out


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

class Clocks:
    def __init__(self, index):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        rows = []
        for r in csv.reader(open(self.path)):
            if len(r) >= 9:
                rows.append([c.strip() for c in r])
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


def fp64_peak_tflops(torch, dev):
    """Measured fp64 tensor throughput of this GPU (cuBLAS DGEMM 8192^3, best
    of 5) -- the roofline denominator for the DMMA kernels (MEASURED_PEAKS.json
    holds no fp64 figure)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    best = 1e9
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best / 1000.0) / 1e12


def int8_peak_tops(torch, dev):
    """Measured int8 tensor throughput (cuBLASLt through torch._int_mm,
    8192^3, best of 5): the roofline denominator of k_oz_gram (the
    MEASURED_PEAKS.json figures are bf16 only).  None if unavailable."""
    n = 8192
    try:
        a = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-64, 64, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
        torch._int_mm(a, b)
        best = 1e9
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best / 1000.0) / 1e12
    except Exception:  # pragma: no cover
        return None


def ozaki_roofline(prof, steps, torch, dev):
    """k_oz_gram (leaf Gram on tcgen05 kind::i8): achieved int8 tensor ops per
    second (every tile x 28 slice products x padded K, counted by the
    library) against the measured int8 GEMM peak."""
    fam = kernel_families(prof)
    if "k_oz_gram" not in fam:
        return None
    cnt, ms, ops = fam["k_oz_gram"]
    achieved = ops / (ms / 1000.0) / 1e12
    peak = int8_peak_tops(torch, dev)
    nominal = 4500.0
    return {"kernel": "k_oz_gram", "bound": "tensor", "achieved": achieved,
            "peak": peak if peak else nominal, "unit": "TOP/s (int8)",
            "frac": achieved / (peak if peak else nominal),
            "frac_of_nominal_4500": achieved / nominal,
            "peak_source": ("int8 cuBLASLt GEMM 8192^3 (torch._int_mm) measured in this run"
                            if peak else "nominal B200 dense int8 4.5 POP/s (no measurement)"),
            "algorithmic_ops_per_launch": ops / cnt, "avg_launch_ms": ms / cnt,
            "launches_per_step": cnt / steps}


STREAMING = ("k_scale_gather", "k_colnorm_part", "k_scale_rows", "k_gather",
             "k_oz_split", "k_oz_split_rows", "k_oz_colmax", "k_oz_rowmax")


def streaming_roofline(prof, prof_bytes, hbm_peak):
    """Factor streaming and truncation kernels (north_star: merge/truncate
    kernels against the HBM peak): achieved = the algorithmic bytes the
    library counts per launch (columns read + written once; digit-plane
    splits: the fp32 block read + 7 int8 planes written) / event-timed
    duration, per kernel and for the family."""
    per = {}
    for key, (cnt, ms, _) in prof.items():
        k = key.rsplit(":", 1)[-1]
        by = prof_bytes.get(key, 0.0)
        if k not in STREAMING or by <= 0.0 or ms <= 0.0:
            continue
        c0, m0, b0 = per.get(k, (0, 0.0, 0.0))
        per[k] = (c0 + cnt, m0 + ms, b0 + by)
    if not per:
        return None
    tb = sum(v[2] for v in per.values())
    tm = sum(v[1] for v in per.values())
    return {"bound": "hbm", "achieved": tb / (tm / 1000.0) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": tb / (tm / 1000.0) / 1e9 / hbm_peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
            "kernels": {k: {"launches": c, "ms": round(m, 4), "algorithmic_gb": round(b / 1e9, 4),
                            "gbs": round(b / (m / 1000.0) / 1e9, 1),
                            "frac": round(b / (m / 1000.0) / 1e9 / hbm_peak, 4)}
                        for k, (c, m, b) in sorted(per.items(), key=lambda t: -t[1][1])}}


def kernel_families(prof, with_overlapped=False):
    """{kernel name: (launches, ms, flops)} summed over phases (the grouped
    DMMA GEMM and its bulk-copy-fed skinny variant form one family)."""
    fam = {}
    for key, (cnt, ms, fl) in prof.items():
        if "/back.prep:" in key and not with_overlapped:
            # launched on the side stream under the bulge chase: their event
            # times include sharing the GPU, so they stay out of the rooflines
            continue
        k = key.rsplit(":", 1)[-1]
        if k == "k_gemm_sk":
            k = "k_gemm"
        c0, m0, f0 = fam.get(k, (0, 0.0, 0.0))
        fam[k] = (c0 + cnt, m0 + ms, f0 + fl)
    return fam


def load_traffic(workload):
    """Measured DRAM bytes per launch of a kernel family (ncu, committed
    under profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {})
    except Exception:
        return {}


def roofline(prof, steps, w, hbm_peak, fp64_peak, prof_bytes=None):
    """Roofline of the kernel family with the largest share of the step.
    k_gemm (the grouped DMMA GEMM: Grams, projections, the two-stage band
    reduction and both back-transforms) is tensor-bound: achieved = its
    algorithmic flops (counted per launch by the library) / its time.
    k_latrd is HBM-bound: algorithmic bytes = the trailing block streamed
    once per column."""
    fam = kernel_families(prof)
    name = max(fam, key=lambda k: fam[k][1])
    cnt, ms, fl = fam[name]
    meas = load_traffic(w.name)
    # a committed measurement applies only to the same launch mix
    # (the ncu launch list counts every launch of the family, overlapped ones too)
    cnt_all = kernel_families(prof, True)[name][0]
    traffic = meas.get(name) if meas.get("launches_per_step") == cnt_all / steps else None
    if name == "k_gemm" and fl > 0:
        peak = fp64_peak()
        achieved = fl / (ms / 1000.0) / 1e12
        return {"kernel": "k_gemm + k_gemm_sk (all DMMA GEMM launches)", "bound": "tensor",
                "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch",
                "peak_source": "fp64 cuBLAS DGEMM 8192^3 measured in this run",
                "algorithmic_flops_per_launch": fl / cnt, "avg_launch_ms": ms / cnt,
                # operands read once + C written (read too when accumulated): what
                # `traffic` (ncu DRAM bytes per launch) is to be compared with
                "algorithmic_bytes_per_launch": (sum(
                    b for k, b in (prof_bytes or {}).items()
                    if k.rsplit(":", 1)[-1] in ("k_gemm", "k_gemm_sk")
                    and "/back.prep:" not in k) / cnt) or None,
                "excluded": "the reflector-only GEMMs overlapped with the bulge chase on the "
                            "side stream (profile keys */back.prep:*)",
                "launches_per_step": cnt / steps, "share": ms / sum(v[1] for v in fam.values())}
    if name == "k_latrd":
        nleaves, q = w.P * w.Q, min(w.c, w.d)
        byts_step = nleaves * 8.0 * sum((q - j - 1) ** 2 for j in range(q - 1))
        achieved = byts_step / ((ms / steps) / 1000.0) / 1e9
        return {"kernel": "k_latrd", "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
                "algorithmic_bytes_per_launch": byts_step / (cnt / steps),
                "avg_launch_ms": ms / cnt}
    return {"kernel": name, "bound": None, "achieved": None, "peak": None, "unit": None,
            "frac": None, "traffic": traffic,
            "note": "latency-bound kernel (no HBM or tensor roofline applies)"}


def run_ours(args, w):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1710_02812_b200 as H
    from paper_1710_02812_b200 import configs
    ctx = H.Context(local)
    cfg = H.MatConfig(gamma=GAMMA, row_block_rows=w.d, col_block_cols=w.c, max_rank=w.k)
    x = configs.generate_torch(w, device=dev)
    row0, m_local = 0, w.m
    if ws > 1:
        # rows sharded by row slice; NCCL communicator for the
        # factor exchanges, id shared through torch.distributed
        uid = [H.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        ctx.init_nccl(rank, ws, uid[0])
        row0, m_local = H.shard_rows(w.m, w.d, rank, ws)
        x = x[row0:row0 + m_local].clone()
        torch.cuda.empty_cache()
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def step(xx, fetch=False):
        if ws > 1:
            return H.rank_k_svd_sharded(xx, w.m, row0, cfg, ctx, fetch=fetch)
        if fetch:
            return H.rank_k_svd(xx, cfg, ctx)
        return H.rank_k_svd_device(xx, cfg, ctx)

    for _ in range(args.warmup):
        step(x)
    ctx.synchronize()
    def timed_pass(profiled):
        """K steps bracketed by barrier + synchronize, timed with CUDA events
        on the library's stream; with per-launch events when profiled."""
        ctx.profile(profiled)
        ctx.profile_report()
        barrier()
        ctx.synchronize()
        torch.cuda.synchronize()
        l0 = ctx.launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            r = step(x)
        e1.record(stream)
        ctx.synchronize()
        torch.cuda.synchronize()
        barrier()
        launches = (ctx.launch_count() - l0) // args.steps
        ms = e0.elapsed_time(e1) / args.steps
        prof = ctx.profile_report() if profiled else None
        ctx.profile(False)
        return r, ms, launches, (prof, dict(ctx.profile_bytes)) if profiled else None

    # timed region (device-resident input): the headline pass runs without
    # per-launch events (they cost ~3% of the step in host launch time); the
    # per-kernel breakdown and the roofline come from a second timed pass of
    # the same K steps with them
    clocks = Clocks(local)
    rank_k, ms, launches, _ = timed_pass(False)
    clk = clocks.stop()
    _, ms_prof, _, (prof, prof_bytes) = timed_pass(True)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = w.input_bytes / (ms / 1000.0) / 1e9  # one matrix per step, whole job

    # e2e through the public API with host buffers (H2D of X, D2H of U, sigma,
    # V): first from pageable memory -- what the C++ drop-in's DenseMatrix
    # (std::vector storage) passes, staged by the library through its pinned
    # ring -- the headline e2e; then from pinned memory (DMA straight from the
    # caller's buffer) as e2e_pinned
    e2e = e2e_pinned = None
    if not args.no_e2e:
        reps = max(1, min(args.steps, 3))

        def time_host(xh):
            step(xh, fetch=True)  # warm
            barrier()
            ctx.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                f = step(xh, fetch=True)
            ctx.synchronize()
            sec = (time.perf_counter() - t0) / reps
            barrier()
            if ws > 1:
                t = torch.tensor([sec], device=dev)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                sec = float(t.item())
            d2h = 8 * (f.u.size + f.v.size + f.sigma.size)
            return {"value": w.input_bytes / sec / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": int(w.input_bytes),
                    "d2h_bytes_per_step": int(d2h) * ws, "ms_per_step": 1000.0 * sec,
                    "timed": f"wall clock over {reps} calls of the public rank_k_svd with "
                             f"host X, results copied back (max over ranks)"}

        xh = x.cpu()
        del x
        torch.cuda.empty_cache()
        e2e = dict(time_host(xh), host_memory="pageable (torch CPU tensor / std::vector "
                                              "storage: the drop-in path)")
        xh = xh.pin_memory()
        e2e_pinned = dict(time_host(xh), host_memory="pinned (cudaHostAlloc)")
        del xh
    if rank != 0:
        return 0

    # kernel shares and roofline of the dominant kernel
    tot = sum(v[1] for v in prof.values()) or 1.0
    shares = sorted(((k, v[0] // args.steps, v[1] / args.steps, v[1] / tot)
                     for k, v in prof.items()), key=lambda t: -t[2])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof = roofline(prof, args.steps, w, hbm_peak, lambda: fp64_peak_tflops(torch, dev), prof_bytes)
    roof["measured"] = ("per-launch CUDA events over a second timed pass of the same K steps "
                        "(the headline pass runs without them)")
    roof["profiled_pass_ms_per_step"] = ms_prof
    oz = ozaki_roofline(prof, args.steps, torch, dev)
    if oz is not None:
        roof["leaf_gram_int8"] = oz
    st = streaming_roofline(prof, prof_bytes, hbm_peak)
    if st is not None:
        roof["factor_streaming_hbm"] = st

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        try:
            cpu = cpu_baseline(args, w)
        except Exception as exc:  # pragma: no cover
            cpu = {"error": str(exc)}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json recipe, generated on device)",
        "config": dict(arm_config(w, ws), rank_out=rank_k),
        "e2e": e2e, "e2e_pinned": e2e_pinned, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
        "clocks": clk,
        "tflops_tc": w.flops_tc() / (ms / 1000.0) / 1e12,
        "kernels": [{"name": k, "launches": n, "ms": round(t, 4), "share": round(s, 4)}
                    for k, n, t, s in shares[:12]],
        "kernels_all": [[k, n, round(t, 4)] for k, n, t, s in shares],
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    ws, _, _ = dist_env()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.launcher_selftest:
        return launcher_selftest(args)
    if args.impl == "ours" and ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    from paper_1710_02812_b200 import configs
    w = configs.WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
