#!/usr/bin/env python
"""Precision study for the int8 Ozaki-sliced block Gram (SURVEY 7.1 step 4,
7.3 H1): how many 7-bit slices does the leaf Gram need so the leaf's top-k
singular values / subspace match the fp64 SVD to well inside the north-star
tolerances?  Exact integer emulation of the tensor-core products (int64
matmul of the int8 digit matrices = the int32 TMEM sums, exact), fp64
recombination, then the same eigen route the device takes (Gram eig +
projection sigma = column norms).

Slicing: per column j, scale_j = 2^e with max_i |x_ij| < scale_j; digit 1 =
rint(x/scale * 64) in [-64, 64], then each next digit = rint(residual * 128)
in [-64, 64].  Products of digits a and b carry weight 2^-(6+7(a-1)) *
2^-(6+7(b-1)); only a + b <= s + 1 are formed (s(s+1)/2 products).
Digit products are summed by fp64 BLAS, exactly (|sum| < 2^31 << 2^53).
"""
import sys

import numpy as np


def split(x, s):
    e = np.ceil(np.log2(np.maximum(np.abs(x).max(axis=0), 1e-300)))
    scale = np.exp2(e)
    r = x / scale
    digits = []
    for a in range(s):
        f = 64.0 if a == 0 else 128.0
        d = np.rint(r * f)
        digits.append(d)
        r = r * f - d
    return digits, scale


def ozaki_gram(x, s):
    digits, scale = split(np.asarray(x, dtype=np.float64), s)
    g = np.zeros((x.shape[1], x.shape[1]))
    for t in range(s + 1, 1, -1):  # least significant level first
        acc = np.zeros_like(g)  # digit products in fp64 BLAS: exact (< 2^53)
        for a in range(1, t):
            b = t - a
            if a > s or b > s:
                continue
            acc += digits[a - 1].T @ digits[b - 1]
        assert np.abs(acc).max() < 2 ** 31
        w = 2.0 ** (-(6 + 7 * (t - 2)) - 6 - 7 * 0)  # 2^-(12 + 7(t-2))
        g += acc * w
    return g * scale[:, None] * scale[None, :]


def leaf_top_k(x, g, k):
    lam, z = np.linalg.eigh(g)
    z = z[:, ::-1][:, :k]
    p = np.asarray(x, dtype=np.float64) @ z
    sig = np.linalg.norm(p, axis=0)
    return sig, p / sig, z


def angle(a, b):
    r = b - a @ (a.T @ b)
    return float(np.arcsin(min(1.0, np.linalg.svd(r, compute_uv=False)[0])))


def case(name, x, k, slices=(3, 4, 5, 6)):
    x64 = np.asarray(x, dtype=np.float64)
    u, s_ref, vt = np.linalg.svd(x64, full_matrices=False)
    u, s_ref, v = u[:, :k], s_ref[:k], vt[:k].T
    print(f"{name}: {x.shape} k={k} sigma_k/sigma_1={s_ref[-1] / s_ref[0]:.2e} "
          f"relgap_k={s_ref[-2] / s_ref[-1] - 1 if k > 1 else 0:.2e}")
    g64 = x64.T @ x64
    sig, uu, z = leaf_top_k(x, g64, k)
    print(f"   fp64 Gram : sigma {np.abs(sig - s_ref).max() / s_ref[-1]:.2e} (rel to sigma_k)  "
          f"angle U {angle(u, uu):.2e} V {angle(v, z):.2e}")
    for s in slices:
        g = ozaki_gram(x, s)
        sig, uu, z = leaf_top_k(x, g, k)
        print(f"   s={s} ({s * (s + 1) // 2:2d} products): |G-G64|/|G| "
              f"{np.abs(g - g64).max() / np.abs(g64).max():.1e}  sigma "
              f"{np.abs(sig - s_ref).max() / s_ref[-1]:.2e}  angle U {angle(u, uu):.2e} "
              f"V {angle(v, z):.2e}")


def lowrank(m, n, r, spec, noise, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    s = spec(np.arange(1, r + 1, dtype=np.float64))
    return ((u * s) @ v.T + noise * rng.standard_normal((m, n))).astype(np.float32)


if __name__ == "__main__":
    sys.path.insert(0, ".")
    from paper_1710_02812_b200 import configs
    # leaves in the shape class of each config, at reduced size (full-matrix
    # spectra scaled so the leaf sees a comparable sigma_k / sigma_1)
    case("cfg2-like leaf", lowrank(2500, 1000, 100, lambda i: i ** -1.5, 1e-3, 2), 100)
    case("cfg5-like leaf", lowrank(2048, 1024, 200, lambda i: 100 * np.exp(-0.05 * i), 1e-4, 5), 200)
    case("cfg3-like leaf", lowrank(8192, 1024, 64, lambda i: np.exp(-0.1 * i), 1e-4, 3), 64)
    w4 = configs.WORKLOADS[4].scaled(16384, 2048, P=1, Q=1)
    x4 = configs.generate_numpy(w4)
    case("cfg4 leaf (modes recipe)", x4[:8192, :1024], 128)
