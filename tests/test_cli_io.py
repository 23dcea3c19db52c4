"""HSVD1 streamed to the device and the `svd` CLI through the C ABI
(SURVEY 8(f) next #3): load_hsvd1's checks and messages
(matrix_io.cpp:91-113), the reference CLI's svd behaviour (test_cli.cpp:56-66:
gen 64x32 rank 4 exp:0.5 seed 7, svd --gamma 1e-6 -> rank 4, sigma
1 0.5 0.25 0.125) and its exit codes (hsvd_main.cpp:27-29)."""
import os
import subprocess

import numpy as np
import pytest

import hsvd_oracle as O
from ref_cases import lowrank

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1710_02812_b200", "hsvd_b200")


def _run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


def test_cli_usage_exit_codes():
    """No GPU needed: usage errors exit 1 before any device call."""
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    assert _run()[0] == 1
    assert _run("--help")[0] == 0
    rc, _, err = _run("svd")
    assert rc == 1 and "--input is required" in err
    rc, _, err = _run("svd", "--input", "x.hsvd", "--gamma", "abc")
    assert rc == 1 and "cannot parse" in err
    assert _run("bogus")[0] == 1


@pytest.mark.gpu
def test_load_hsvd1_roundtrip_and_errors(tmp_path):
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(9)
    x = rng.standard_normal((300, 70))
    p = str(tmp_path / "x.hsvd")
    H.save_hsvd1(x, p)
    dm = H.load_hsvd1(p)
    assert dm.shape == (300, 70)
    f = H.rank_k_svd(dm, H.MatConfig(gamma=0.0, row_block_rows=100, col_block_cols=35))
    assert np.abs(f.sigma - O.full_svd(x).sigma).max() < 1e-10 * O.full_svd(x).sigma[0]
    # the reference's error cases and messages
    with pytest.raises(H.IoError, match="cannot open for reading"):
        H.load_hsvd1(str(tmp_path / "missing.hsvd"))
    bad = tmp_path / "bad.hsvd"
    bad.write_bytes(b"HSVD2\0" + bytes(16))
    with pytest.raises(H.FormatError, match="bad magic"):
        H.load_hsvd1(str(bad))
    short = tmp_path / "short.hsvd"
    short.write_bytes(b"HSVD1\0" + bytes(5))
    with pytest.raises(H.FormatError, match="truncated header"):
        H.load_hsvd1(str(short))
    empty = tmp_path / "empty.hsvd"
    empty.write_bytes(b"HSVD1\0" + (0).to_bytes(8, "little") + (3).to_bytes(8, "little"))
    with pytest.raises(H.FormatError, match="empty matrix"):
        H.load_hsvd1(str(empty))
    huge = tmp_path / "huge.hsvd"
    huge.write_bytes(b"HSVD1\0" + (1 << 40).to_bytes(8, "little") + (2).to_bytes(8, "little"))
    with pytest.raises(H.FormatError, match="implausible dimensions"):
        H.load_hsvd1(str(huge))
    trunc = tmp_path / "trunc.hsvd"
    trunc.write_bytes(b"HSVD1\0" + (4).to_bytes(8, "little") + (4).to_bytes(8, "little") +
                      bytes(8 * 10))
    with pytest.raises(H.FormatError, match="truncated payload"):
        H.load_hsvd1(str(trunc))
    nan = x.copy()
    nan[17, 3] = np.nan
    H.save_hsvd1(nan, str(tmp_path / "nan.hsvd"))
    with pytest.raises(H.FormatError, match="NaN or Inf"):
        H.load_hsvd1(str(tmp_path / "nan.hsvd"))


@pytest.mark.gpu
def test_cli_svd_matches_reference_cli(tmp_path, golden):
    x, _ = lowrank(golden, 64, 32, 7, "exp", 4, ratio=0.5)
    import paper_1710_02812_b200 as H
    p = str(tmp_path / "x.hsvd")
    H.save_hsvd1(x, p)
    rc, out, err = _run("svd", "--input", p, "--gamma", "1e-6", "--precise",
                        "--out-prefix", str(tmp_path / "f"))
    assert rc == 0, err
    lines = out.splitlines()
    assert lines[0] == "rank 4"
    sig = [float(t) for t in lines[1].split()[1:]]
    assert np.allclose(sig, [1.0, 0.5, 0.25, 0.125], rtol=1e-10, atol=0)
    s_csv = np.loadtxt(str(tmp_path / "f_sigma.csv"))
    assert np.allclose(s_csv, sig, rtol=0, atol=0)
    u = H.load_hsvd1(str(tmp_path / "f_U.hsvd"))
    assert u.shape == (64, 4)
    # refinement and the rank cap
    rc, out, err = _run("svd", "--input", p, "--gamma", "1e-6", "--refine", "--eps", "1e-8")
    assert rc == 0 and out.startswith("refined in "), err
    rc, out, err = _run("svd", "--input", p, "--gamma", "1e-6", "--max-rank", "2")
    assert rc == 0 and out.splitlines()[0] == "rank 2", err
    rc, _, err = _run("svd", "--input", str(tmp_path / "none.hsvd"))
    assert rc == 2 and "cannot open for reading" in err


@pytest.mark.gpu
def test_fp32_payload_variant(tmp_path):
    """HSVF1: the fp32 payload variant (half the bytes of HSVD1) loads to an
    fp32 device matrix and decomposes to the same factors as the fp32 host
    input; the fp64-only load_hsvd1 keeps the reference's behaviour (bad
    magic); the CLI reads either form."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(32)
    x = rng.standard_normal((400, 96)).astype(np.float32)
    p = str(tmp_path / "x32.hsvd")
    H.save_hsvd1(x, p, dtype="f32")
    assert os.path.getsize(p) == 22 + 4 * x.size
    dm = H.load_matrix(p)
    assert dm.shape == (400, 96) and dm.dtype == H.hsvd.F32
    cfg = H.MatConfig(gamma=0.0, row_block_rows=100, col_block_cols=48, max_rank=20)
    a = H.rank_k_svd(dm, cfg)
    b = H.rank_k_svd(x, cfg)
    assert np.array_equal(a.sigma, b.sigma)
    with pytest.raises(H.FormatError, match="bad magic"):
        H.load_hsvd1(p)
    d64 = str(tmp_path / "x64.hsvd")
    H.save_hsvd1(x.astype(np.float64), d64)
    assert H.load_matrix(d64).dtype == H.hsvd.F64
    bad = x.copy()
    bad[5, 5] = np.inf
    H.save_hsvd1(bad, str(tmp_path / "inf32.hsvd"), dtype="f32")
    with pytest.raises(H.FormatError, match="NaN or Inf"):
        H.load_matrix(str(tmp_path / "inf32.hsvd"))
    rc, out, err = _run("svd", "--input", p, "--gamma", "0", "--row-block", "100",
                        "--col-block", "48", "--max-rank", "20", "--precise")
    assert rc == 0, err
    sig = [float(t) for t in out.splitlines()[1].split()[1:]]
    assert out.splitlines()[0] == "rank 20"
    assert np.allclose(sig, a.sigma[:len(sig)], rtol=1e-12, atol=0)
