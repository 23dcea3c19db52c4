"""Generate tests/golden/ref_gaussians.npz (TEST INFRASTRUCTURE ONLY).

Builds ``oracle/gen_ref_gaussians.cpp`` with g++ into ``oracle/_bin/`` and
records the reference's seeded Gaussian streams for every fixture the
known-answer tests need (see tests/test_oracle_golden.py for the reference
file:line each one comes from).  Re-run with ``python oracle/make_golden.py``.
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
BIN = os.path.join(HERE, "_bin", "gen_ref_gaussians")
OUT = os.path.join(ROOT, "tests", "golden", "ref_gaussians.npz")


def build() -> str:
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    src = os.path.join(HERE, "gen_ref_gaussians.cpp")
    if (not os.path.exists(BIN)) or os.path.getmtime(BIN) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-std=c++17", src, "-o", BIN])
    return BIN


def specs():
    """(key, kind, a, b, seed) for every fixture."""
    out = []
    # generator cases: (m, n, seed)
    for m, n, seed in [(64, 32, 2024), (64, 32, 7), (256, 64, 620), (16, 8, 77),
                       (40, 20, 9), (512, 128, 820),
                       # test_bench.cpp sharp_decay_matrix fixtures
                       (64, 32, 4000), (96, 48, 4100), (32, 16, 4200), (16, 8, 4300),
                       (48, 24, 4400), (32, 16, 4500), (16, 8, 4600), (16, 8, 4700)]:
        out.append((f"lr_{m}x{n}_s{seed}", "lowrank", m, n, seed))
    # random_matrix cases used by test_hierarchy / test_kernels / test_merge
    mats = [(48, 32, 630), (40, 64, 456), (40, 16, 10000), (60, 30, 640),
            (30, 14, 650), (12, 12, 660), (50, 20, 670), (24, 10, 610),
            (16, 8, 510), (10, 6, 680), (20, 6, 51), (20, 6, 52), (5, 14, 53),
            (7, 14, 54), (10, 3, 55), (14, 9, 5), (5, 3, 7)]
    # acceptance.cpp:77-112 exactness matrices
    for t in range(20):
        mats.append((40 + 8 * (t % 21), 16 + 8 * (t % 7), 10000 + t))
    # test_kernels.cpp:108-122 Gram-oracle sizes
    for n in (8, 16, 31, 32, 33, 48):
        mats.append((2 * n, n, 5000 + n))
    # test_merge.cpp:126-155: random_factor bases (u for column trials, v for row)
    for t in range(100):
        m = 8 + t % 23
        k = 1 + t % 5
        l = 1 + (t * 3) % 5
        if t % 2 == 0:
            mats += [(m, k, 1000 + 7 * t), (m, l, 2000 + 7 * t)]
        else:
            mats += [(m, k, 1001 + 7 * t), (m, l, 2001 + 7 * t)]
    # acceptance.cpp:115-149 merge oracle
    for t in range(100):
        shared = 10 + t % 41
        k = 1 + t % 6
        l = 1 + (t * 5) % 6
        mats += [(shared, k, 20000 + 4 * t), (shared, l, 20001 + 4 * t),
                 (shared, k, 20002 + 4 * t), (shared, l, 20003 + 4 * t)]
    # test_merge.cpp property tests (random_factor(m, n, k, seed) -> u seed, v seed+1)
    for t in range(20):
        mats += [(15, 3, 3000 + t), (15, 4, 4000 + t), (18, 4, 5000 + t),
                 (18, 5, 6000 + t), (16, 3, 7000 + t), (16, 5, 8000 + t)]
    mats += [(12, 3, 9100), (12, 3, 9200), (12, 4, 9300), (12, 4, 9400),
             (5, 4, 9500), (5, 4, 9600), (10, 1, 9700), (10, 3, 9800)]
    # test_refine.cpp
    mats += [(24, 12, 800), (30, 15, 810), (5, 5, 811), (40, 18, 830), (50, 25, 840),
             (30, 20, 860), (20, 10, 870), (10, 6, 880), (6, 2, 881)]
    for t in range(50):
        mats.append((24 + 4 * (t % 5), 12 + 2 * (t % 4), 850 + t))
    seen = set()
    for r, c, s in mats:
        key = f"m_{r}x{c}_s{s}"
        if key in seen:
            continue
        seen.add(key)
        out.append((key, "matrix", r, c, s))
    return out


def main() -> int:
    exe = build()
    sp = specs()
    text = "".join(f"{kind} {a} {b} {seed}\n" for _k, kind, a, b, seed in sp)
    raw = subprocess.run([exe], input=text.encode(), stdout=subprocess.PIPE,
                         check=True).stdout
    buf = np.frombuffer(raw, dtype="<f8")
    arrays = {}
    off = 0
    for key, kind, a, b, _seed in sp:
        if kind == "matrix":
            n = a * b
            arrays[key] = buf[off:off + n].reshape(a, b).copy()
            off += n
        else:
            p = min(a, b)
            arrays[key + "_gu"] = buf[off:off + a * p].reshape(a, p).copy()
            off += a * p
            arrays[key + "_gv"] = buf[off:off + b * p].reshape(b, p).copy()
            off += b * p
    assert off == buf.shape[0], (off, buf.shape)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {len(arrays)} arrays ({buf.nbytes} bytes) to {OUT}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
