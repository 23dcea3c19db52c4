"""Benchmark report with GPU timings: the reference's
test_bench.cpp restated (run_benchmark on the device; JSON schema checks;
cost model), with the sharp-decay fixtures of test_bench.cpp:11-20 from the
golden Gaussian streams."""
import json

import numpy as np
import pytest

import hsvd_oracle as O
from ref_cases import lowrank


def _sharp(golden, m, n, seed):
    """test_bench.cpp:11-20: gen_low_rank exp ratio 0.5, rank 8, floor 1e-8."""
    return lowrank(golden, m, n, seed, "exp", 8, ratio=0.5, floor=1e-8)[0]


def _sample_report():
    from paper_1710_02812_b200 import report as R
    rep = R.BenchReport(rows=32, cols=16, gamma=1e-2, epsilon=1e-3, repeats=1,
                        kernel_threads=148)
    rep.entries.append(R.BenchEntry(block_rows=-1, block_cols=4, error="bad plan"))
    rep.entries.append(R.BenchEntry(block_rows=32, block_cols=16, recovered_rank=3,
                                    wall_time_mat_s=0.5, wall_time_full_svd_s=1.0, speedup=2.0,
                                    rel_error=1e-12, sigma_head=[1.0, 0.5, 0.25],
                                    predicted=R.estimate_costs(32, 16, 1, 3),
                                    wall_time_mat_refined_s=0.6, speedup_refined=1.0 / 0.6,
                                    rel_error_refined=1e-13))
    return rep


def test_cost_model_formulas():
    """cost_model.hpp:22-60."""
    from paper_1710_02812_b200 import report as R
    assert R.flops_full_svd(100, 10) == 6 * 100 * 100 + 16 * 1000
    with pytest.raises(ValueError):
        R.flops_full_svd(10, 100)
    s = 40 / 4
    assert R.flops_mat_partition(100, 40, 4, 5) == pytest.approx(
        4 * (6 * 100 * s * s + 16 * s ** 3) + 3 * (14 * 100 * 25 + 176 * 125))
    with pytest.raises(ValueError):
        R.flops_mat_partition(100, 40, 4, 11)  # k > s
    assert R.speedup_bound(100, 40, 4) == pytest.approx(20 * 100 * 1600 / 4 + 192 * 64000 / 16)
    est = R.estimate_costs(16, 32, 2, 4)  # wide: full SVD in the tall orientation
    assert est.flops_full == R.flops_full_svd(32, 16) and est.partitions == 2


def test_report_json_schema_round_trip_and_mutations():
    """test_bench.cpp:80-121 (on a hand-built report: no GPU needed)."""
    from paper_1710_02812_b200 import report as R
    good = R.report_to_json(_sample_report())
    assert R.validate_report_json(good) == []
    assert '"error"' in good
    assert R.validate_report_json("{ not json") != []
    assert R.validate_report_json("[]") != []
    assert R.validate_report_json("{}") != []
    assert R.validate_report_json(good.replace('"gamma"', '"gamme"', 1)) != []
    doc = json.loads(good)
    doc["grid"][1]["recovered_rank"] = "3"
    assert R.validate_report_json(json.dumps(doc)) != []
    doc = json.loads(good)
    del doc["grid"][1]["speedup_refined"]  # refined metrics must come together
    assert R.validate_report_json(json.dumps(doc)) != []
    doc = json.loads(good)
    doc["grid"][1]["sigma_head"] = [0.0] * 65
    assert R.validate_report_json(json.dumps(doc)) != []


@pytest.mark.gpu
def test_run_benchmark_single_block(golden):
    """test_bench.cpp:23-41."""
    import paper_1710_02812_b200 as H
    from paper_1710_02812_b200 import report as R
    x = _sharp(golden, 64, 32, 4000)
    rep = R.run_benchmark(x, H.MatConfig(gamma=1e-2), [R.GridPoint(64, 32)], 2, False)
    assert len(rep.entries) == 1
    e = rep.entries[0]
    assert e.error == ""
    assert e.rel_error <= 1e-10
    assert e.recovered_rank >= 1
    assert e.wall_time_mat_s > 0.0 and e.wall_time_full_svd_s > 0.0
    assert e.speedup == pytest.approx(e.wall_time_full_svd_s / e.wall_time_mat_s, rel=1e-12)
    assert e.wall_time_mat_refined_s is None
    assert len(e.sigma_head) == e.recovered_rank
    assert e.predicted is not None and e.predicted.partitions == 1


@pytest.mark.gpu
def test_run_benchmark_refined_never_lose(golden):
    """test_bench.cpp:43-59."""
    import paper_1710_02812_b200 as H
    from paper_1710_02812_b200 import report as R
    x = _sharp(golden, 96, 48, 4100)
    grid = [R.GridPoint(96, 48), R.GridPoint(48, 12), R.GridPoint(24, 8)]
    rep = R.run_benchmark(x, H.MatConfig(gamma=1e-2), grid, 1, True)
    assert len(rep.entries) == 3
    for e in rep.entries:
        assert e.error == ""
        assert e.rel_error_refined <= e.rel_error + 1e-12
        assert e.speedup_refined == pytest.approx(e.wall_time_full_svd_s /
                                                  e.wall_time_mat_refined_s, rel=1e-12)


@pytest.mark.gpu
def test_run_benchmark_failures_and_arguments(golden):
    """test_bench.cpp:61-78, 114-131."""
    import paper_1710_02812_b200 as H
    from paper_1710_02812_b200 import report as R
    x = _sharp(golden, 32, 16, 4200)
    rep = R.run_benchmark(x, H.MatConfig(gamma=1e-2), [R.GridPoint(-3, -3), R.GridPoint(32, 16)],
                          1, False)
    assert rep.entries[0].error != "" and rep.entries[1].error == ""
    x = _sharp(golden, 16, 8, 4300)
    with pytest.raises(ValueError):
        R.run_benchmark(x, H.MatConfig(), [], 1, False)
    with pytest.raises(ValueError):
        R.run_benchmark(x, H.MatConfig(), [R.GridPoint(16, 8)], 0, False)
    x = _sharp(golden, 16, 8, 4600)
    text = R.report_to_json(R.run_benchmark(x, H.MatConfig(), [R.GridPoint(-1, 4),
                                                             R.GridPoint(16, 8)], 1, False))
    assert R.validate_report_json(text) == [] and '"error"' in text
    x = _sharp(golden, 16, 8, 4700)
    rep = R.run_benchmark(x, H.MatConfig(), [R.GridPoint(16, 8)], 1, False)
    assert rep.kernel_threads >= 1 and rep.repeats == 1 and rep.rows == 16 and rep.cols == 8
    x = _sharp(golden, 48, 24, 4400)
    rep = R.run_benchmark(x, H.MatConfig(gamma=1e-2), [R.GridPoint(48, 24), R.GridPoint(24, 6)],
                          1, True)
    assert R.validate_report_json(R.report_to_json(rep)) == []


@pytest.mark.gpu
def test_report_cli_writes_valid_json(tmp_path, golden):
    """The `bench` subcommand (hsvd_main.cpp:161-190) as a module entry point."""
    import paper_1710_02812_b200 as H
    from paper_1710_02812_b200 import report as R
    x = _sharp(golden, 96, 48, 4100)
    p = str(tmp_path / "x.hsvd")
    H.save_hsvd1(x, p)
    out = str(tmp_path / "r.json")
    assert R.main(["--input", p, "--grid", "96x48,48x12", "--repeats", "1", "--refine",
                   "--json", out]) == 0
    assert R.validate_report_json(open(out).read()) == []
    assert R.main(["--input", p, "--grid", "96y48"]) == 1
    assert R.main(["--input", str(tmp_path / "none.hsvd"), "--grid", "8x8"]) == 2
