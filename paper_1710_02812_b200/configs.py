"""The five BASELINE.json workloads and their seeded synthetic generators.

There is no public dataset for this path (the paper's CFD/FACES data is not
available); each config is generated from the recipe in BASELINE.json:
X = U diag(s) V^T + sigma_N * N with U, V orthonormal (QR of seeded Gaussians,
formed in fp64, then rounded to the config dtype), or, for config 4, a sum of
128 separable sin/cos modes with power-law amplitudes.  Spectra are 1-based
(i = 1..r).  The generator runs on the GPU with torch (input preparation, not
part of the timed path) or on the CPU with numpy for reduced sizes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

SEED_BASE = 171002812


@dataclass(frozen=True)
class Workload:
    cfg: int
    m: int
    n: int
    dtype: str          # "f32" | "f64"
    P: int
    Q: int
    k: int
    kind: str           # "lowrank" | "modes"
    r: int
    noise: float
    spectrum: Callable[[np.ndarray], np.ndarray]

    @property
    def d(self) -> int:
        return self.m // self.P

    @property
    def c(self) -> int:
        return self.n // self.Q

    @property
    def itemsize(self) -> int:
        return 4 if self.dtype == "f32" else 8

    @property
    def input_bytes(self) -> int:
        return self.m * self.n * self.itemsize

    @property
    def name(self) -> str:
        return (f"cfg{self.cfg}_{self.m}x{self.n}_{self.dtype}_grid{self.P}x{self.Q}_k{self.k}")

    def scaled(self, m: int, n: int, P: int = None, Q: int = None, k: int = None) -> "Workload":
        return Workload(self.cfg, m, n, self.dtype, P or self.P, Q or self.Q, k or self.k,
                        self.kind, min(self.r, m, n), self.noise, self.spectrum)

    def flops_tc(self) -> float:
        """F_tc = 2 m n c + 6 m n k (block Grams + leaf
        projection + V-recovery + U-recovery)."""
        return 2.0 * self.m * self.n * min(self.c, self.d) + 6.0 * self.m * self.n * self.k


WORKLOADS = {
    1: Workload(1, 2000, 2000, "f64", 4, 4, 50, "lowrank", 50, 1e-4,
                lambda i: 10.0 * np.exp(-0.15 * i)),
    2: Workload(2, 20000, 20000, "f32", 8, 8, 100, "lowrank", 100, 1e-3,
                lambda i: i ** -1.5),
    3: Workload(3, 1048576, 2048, "f32", 64, 1, 64, "lowrank", 64, 1e-4,
                lambda i: np.exp(-0.1 * i)),
    4: Workload(4, 262144, 8192, "f32", 16, 4, 128, "modes", 128, 1e-3,
                lambda i: i ** -2.0),
    5: Workload(5, 65536, 65536, "f32", 16, 16, 200, "lowrank", 200, 1e-4,
                lambda i: 100.0 * np.exp(-0.05 * i)),
}


def _mode_params(w: Workload, rng):
    t = np.arange(1, w.r + 1, dtype=np.float64)
    a = rng.uniform(1.0, 32.0, w.r)
    b = rng.uniform(1.0, 16.0, w.r)
    al = rng.uniform(0.0, 2 * math.pi, w.r)
    be = rng.uniform(0.0, 2 * math.pi, w.r)
    return t, a, b, al, be


def generate_numpy(w: Workload, seed: int = None) -> np.ndarray:
    """CPU generator (reduced sizes)."""
    seed = SEED_BASE + w.cfg if seed is None else seed
    rng = np.random.default_rng(seed)
    if w.kind == "modes":
        t, a, b, al, be = _mode_params(w, rng)
        i = np.arange(w.m, dtype=np.float64)[:, None]
        j = np.arange(w.n, dtype=np.float64)[:, None]
        ph = 2 * math.pi * a[None, :] * i / w.m + al[None, :]
        phi = np.where((np.arange(w.r) % 2 == 0)[None, :], np.sin(ph), np.cos(ph))
        psi = np.cos(2 * math.pi * b[None, :] * j / w.n + be[None, :])
        x = (phi * w.spectrum(t)) @ psi.T
    else:
        u = np.linalg.qr(rng.standard_normal((w.m, w.r)))[0]
        v = np.linalg.qr(rng.standard_normal((w.n, w.r)))[0]
        s = w.spectrum(np.arange(1, w.r + 1, dtype=np.float64))
        x = (u * s) @ v.T
    x += w.noise * rng.standard_normal((w.m, w.n))
    return x.astype(np.float32 if w.dtype == "f32" else np.float64)


def generate_torch(w: Workload, device="cuda", seed: int = None, chunk_rows: int = 4096):
    """GPU generator for full-size configs (fp64 assembly, rounded once)."""
    import torch
    seed = SEED_BASE + w.cfg if seed is None else seed
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    f64 = torch.float64
    out_dt = torch.float32 if w.dtype == "f32" else torch.float64
    x = torch.empty((w.m, w.n), dtype=out_dt, device=device)
    if w.kind == "modes":
        rng = np.random.default_rng(seed)
        t, a, b, al, be = _mode_params(w, rng)
        amp = torch.tensor(w.spectrum(t), dtype=f64, device=device)
        a_t = torch.tensor(a, dtype=f64, device=device)
        b_t = torch.tensor(b, dtype=f64, device=device)
        al_t = torch.tensor(al, dtype=f64, device=device)
        be_t = torch.tensor(be, dtype=f64, device=device)
        even = (torch.arange(w.r, device=device) % 2 == 0)
        j = torch.arange(w.n, dtype=f64, device=device)[:, None]
        psi = torch.cos(2 * math.pi * b_t[None, :] * j / w.n + be_t[None, :])
        left_scale = amp
        right = psi
        def left_rows(r0, r1):
            i = torch.arange(r0, r1, dtype=f64, device=device)[:, None]
            ph = 2 * math.pi * a_t[None, :] * i / w.m + al_t[None, :]
            return torch.where(even[None, :], torch.sin(ph), torch.cos(ph)) * left_scale
    else:
        u = torch.linalg.qr(torch.randn((w.m, w.r), dtype=f64, device=device, generator=g))[0]
        v = torch.linalg.qr(torch.randn((w.n, w.r), dtype=f64, device=device, generator=g))[0]
        s = torch.tensor(w.spectrum(np.arange(1, w.r + 1, dtype=np.float64)), dtype=f64,
                         device=device)
        u = u * s
        right = v
        def left_rows(r0, r1):
            return u[r0:r1]
    for r0 in range(0, w.m, chunk_rows):
        r1 = min(w.m, r0 + chunk_rows)
        blk = left_rows(r0, r1) @ right.T
        blk += w.noise * torch.randn((r1 - r0, w.n), dtype=f64, device=device, generator=g)
        x[r0:r1] = blk.to(out_dt)
        del blk
    return x
