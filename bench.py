#!/usr/bin/env python
"""Benchmark of the rank-k HSVD hot path (hierarchical_svd + recover_left_vectors).

Metric (BASELINE.json): HSVD input GB/s = m*n*sizeof(dtype) / t per rank-k
SVD, whole job.  One step = one full rank-k HSVD of the workload matrix.
Default workload: BASELINE config 2 (20000x20000 fp32, 8x8 grid, k=100).

  python bench.py [--gpus N --steps K --warmup W --config C]
  python bench.py --impl reference ...   (CPU oracle arm, rank 0 only)

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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU arm (oracle port on the host cores)
# ---------------------------------------------------------------------------

def cpu_slice_sample(w, threads):
    """Row slice 0 of workload w through the CPU oracle: its Q leaf SVDs,
    column merges and V-recovery (1/P of the leaf work).  Returns
    (seconds, slice bytes, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import hsvd_oracle as O
    from paper_1710_02812_b200 import configs
    rng = np.random.default_rng(configs.SEED_BASE + w.cfg)
    d = w.d
    if w.kind == "modes":
        full = configs.generate_numpy(w.scaled(d, w.n, P=1), seed=configs.SEED_BASE + w.cfg)
        xs = full
    else:
        u = np.linalg.qr(rng.standard_normal((w.m, w.r)))[0][:d]
        v = np.linalg.qr(rng.standard_normal((w.n, w.r)))[0]
        s = w.spectrum(np.arange(1, w.r + 1, dtype=np.float64))
        xs = (u * s) @ v.T + w.noise * rng.standard_normal((d, w.n))
        xs = xs.astype(np.float32 if w.dtype == "f32" else np.float64)
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    t0 = time.perf_counter()
    if threadpool_limits is not None and threads > 1 and w.Q > 1:
        with threadpool_limits(1):
            um = O.svd_of_col_slices(xs, w.c, GAMMA, w.k, workers=threads)
    else:
        um = O.svd_of_col_slices(xs, w.c, GAMMA, w.k, workers=1)
    rec = O.full_svd(um.u.T @ xs.astype(np.float64))
    O.truncate_factor(rec, GAMMA, w.k)
    sec = time.perf_counter() - t0
    desc = (f"row slice 0 of {w.P} ({d}x{w.n}): {w.Q} leaf SVDs + {w.Q - 1} column merges + "
            f"V-recovery, numpy/LAPACK oracle, {threads} threads")
    return sec, xs.nbytes, desc


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
    times = []
    sample_bytes = 0
    desc = ""
    for i in range(args.warmup + args.steps):
        sec, sample_bytes, desc = cpu_slice_sample(w, threads)
        if i >= args.warmup:
            times.append(sec)
    ms = 1000.0 * statistics.mean(times)
    value = sample_bytes / (ms / 1000.0) / 1e9
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


def kernel_families(prof):
    """{kernel name: (launches, ms, flops)} summed over phases."""
    fam = {}
    for key, (cnt, ms, fl) in prof.items():
        k = key.rsplit(":", 1)[-1]
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


def roofline(prof, steps, w, hbm_peak, fp64_peak):
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
    traffic = meas.get(name) if meas.get("launches_per_step") == cnt / steps else None
    if name == "k_gemm" and fl > 0:
        peak = fp64_peak()
        achieved = fl / (ms / 1000.0) / 1e12
        return {"kernel": "k_gemm (all launches)", "bound": "tensor", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "bytes per launch",
                "peak_source": "fp64 cuBLAS DGEMM 8192^3 measured in this run",
                "algorithmic_flops_per_launch": fl / cnt, "avg_launch_ms": ms / cnt,
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
        return r, ms, launches, prof

    # timed region (device-resident input): the headline pass runs without
    # per-launch events (they cost ~3% of the step in host launch time); the
    # per-kernel breakdown and the roofline come from a second timed pass of
    # the same K steps with them
    clocks = Clocks(local)
    rank_k, ms, launches, _ = timed_pass(False)
    clk = clocks.stop()
    _, ms_prof, _, prof = timed_pass(True)
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = w.input_bytes / (ms / 1000.0) / 1e9  # one matrix per step, whole job

    # e2e through the public API with host buffers (H2D of X, D2H of U, sigma, V)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        del x
        torch.cuda.empty_cache()
        step(xh, fetch=True)  # warm
        barrier()
        ctx.synchronize()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 3))):
            f = step(xh, fetch=True)
        ctx.synchronize()
        sec = (time.perf_counter() - t0) / max(1, min(args.steps, 3))
        barrier()
        if ws > 1:
            t = torch.tensor([sec], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            sec = float(t.item())
        d2h = 8 * (f.u.size + f.v.size + f.sigma.size)
        e2e = {"value": w.input_bytes / sec / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(w.input_bytes), "d2h_bytes_per_step": int(d2h) * ws,
               "ms_per_step": 1000.0 * sec}
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
    roof = roofline(prof, args.steps, w, hbm_peak, lambda: fp64_peak_tflops(torch, dev))
    roof["measured"] = ("per-launch CUDA events over a second timed pass of the same K steps "
                        "(the headline pass runs without them)")
    roof["profiled_pass_ms_per_step"] = ms_prof

    cpu = None
    if not args.no_cpu_baseline and ws == 1:
        try:
            threads = args.cpu_threads or os.cpu_count() or 1
            sec, sb, desc = cpu_slice_sample(w, threads)
            cpu = {"value": sb / sec / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
                   "sample": desc, "seconds": sec}
        except Exception as exc:  # pragma: no cover
            cpu = {"error": str(exc)}

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE.json recipe, generated on device)",
        "config": dict(arm_config(w, ws), rank_out=rank_k),
        "e2e": e2e, "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu,
        "clocks": clk,
        "tflops_tc": w.flops_tc() / (ms / 1000.0) / 1e12,
        "kernels": [{"name": k, "launches": n, "ms": round(t, 4), "share": round(s, 4)}
                    for k, n, t, s in shares[:12]],
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    from paper_1710_02812_b200 import configs
    w = configs.WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
