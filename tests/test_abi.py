"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/hsvd_cu.h declares, validates configs like the reference, and
fails loudly (no CPU fallback) when no device is present."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    import paper_1710_02812_b200 as H
    return H, H.load_library()


def test_exports_every_declared_symbol():
    H, lib = _lib()
    hdr = open(os.path.join(ROOT, "include", "hsvd_cu.h")).read()
    declared = sorted(set(re.findall(r"\b(hsvd_cu_[a-z0-9_]+)\s*\(", hdr)))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(H.EXPORTED) == declared


def test_validate_matches_reference():
    H, lib = _lib()
    ok = H.MatConfig()._c()
    assert lib.hsvd_cu_validate(ctypes.byref(ok)) == 0
    for bad in (dict(gamma=-0.1), dict(epsilon=0.0), dict(max_iters=0), dict(max_rank=0),
                dict(row_block_rows=-1)):
        cfg = H.MatConfig(**bad)
        with pytest.raises(ValueError):
            H.validate(cfg)
        c = cfg._c()
        if bad.get("max_rank") == 0:
            continue  # 0 means "no cap" at the C boundary; None-vs-0 is a host-side check
        assert lib.hsvd_cu_validate(ctypes.byref(c)) == H.hsvd.EINVAL


def test_no_cpu_fallback_without_device():
    H, lib = _lib()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(H.HsvdCudaError):
        H.Context(0)


def test_host_logic_matches_oracle():
    import numpy as np
    import hsvd_oracle as O
    H, _ = _lib()
    for ext in (1, 7, 10, 64):
        for blk in (0, 1, 3, 4, 64, 99):
            assert H.partition(ext, blk) == O.partition(ext, blk)
    rng = np.random.default_rng(5)
    for _ in range(200):
        s = np.sort(rng.random(rng.integers(1, 9)))[::-1]
        g = float(rng.random()) if rng.random() > 0.2 else 0.0
        assert H.retained_count(s, g) == O.retained_count(s, g)
    assert H.retained_count(np.zeros(3), 0.5) == 1
