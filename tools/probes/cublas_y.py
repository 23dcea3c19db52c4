"""Probe: cuBLAS (torch.bmm, fp64) time for the stage-1 shapes of config 5 / 2
(Y = A22 V, m x m times m x 32, batched) and the SYR2K-as-GEMM (m x 256 x m)."""
import torch
import time

def t(f, reps=5):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for (b, m) in [(256, 4064), (256, 2048), (256, 1024), (64, 2468), (64, 1200)]:
    A = torch.randn(b, m, m, dtype=torch.float64, device="cuda")
    V = torch.randn(b, m, 32, dtype=torch.float64, device="cuda")
    ms = t(lambda: torch.bmm(A, V))
    fl = 2.0 * b * m * m * 32
    W = torch.randn(b, m, 256, dtype=torch.float64, device="cuda")
    ms2 = t(lambda: torch.baddbmm(A, W, W.transpose(1, 2), alpha=-1.0))
    fl2 = 2.0 * b * m * m * 256
    print(f"b={b} m={m}: Y {ms:.2f} ms {fl/ms/1e9:.1f} TF/s; full GEMM K=256 {ms2:.2f} ms {fl2/ms2/1e9:.1f} TF/s (SYR2K-equivalent {fl2/2/ms2/1e9:.1f})", flush=True)
    del A, V, W
    torch.cuda.empty_cache()
