"""The drop-in benchmark harness (paper_2207_09334_b200.benchmark) against the
reference's own tests of springsim.bench (tests/test_bench.py:17-104)."""

import pytest

import paper_2207_09334_b200.benchmark as bench
from paper_2207_09334_b200.benchmark import (BenchReport, block_cells, block_scene, block_springs, profile,
                                             profile_table, run_bench)


@pytest.mark.parametrize("cells", [1, 2, 3])
def test_spring_formula_matches_builder(cells):
    scene = block_scene(cells)
    assert scene.spring_count == block_springs(cells)
    assert scene.mass_count == (cells + 1) ** 3


@pytest.mark.parametrize("target", [28, 500, 10_000, 100_000, 1_000_000])
def test_block_cells_minimizes_distance(target):
    chosen = block_cells(target)
    best = min(range(1, 60), key=lambda n: abs(block_springs(n) - target))
    assert abs(block_springs(chosen) - target) == abs(block_springs(best) - target)


def test_short_measurements_rejected():
    with pytest.raises(ValueError, match="steps must be >= 100"):
        run_bench(3000, steps=99)


def test_report_invariants_enforced():
    with pytest.raises(ValueError, match="steps"):
        BenchReport(device="d", spring_count=1, mass_count=1, steps=10, wall_time=1.0, throughput=1.0,
                    threads=1, integrator="euler", mode="serial")
    with pytest.raises(ValueError, match="throughput"):
        BenchReport(device="d", spring_count=1, mass_count=1, steps=100, wall_time=1.0, throughput=0.0,
                    threads=1, integrator="euler", mode="serial")


def test_memory_failure_names_the_attempted_size(monkeypatch):
    def boom(cells):
        raise MemoryError
    monkeypatch.setattr(bench, "block_scene", boom)
    with pytest.raises(RuntimeError, match="out of memory.*spring"):
        run_bench(10_000)


@pytest.mark.gpu
def test_report_fields():
    report = run_bench(3000, steps=100, integrator="euler", mode="serial")
    assert report.steps == 100 and report.throughput > 0.0 and report.wall_time > 0.0
    assert report.threads >= 1 and report.integrator == "euler"
    assert report.spring_count == block_springs(block_cells(3000))
    assert report.throughput == pytest.approx(report.spring_count * report.steps / report.wall_time)


@pytest.mark.gpu
def test_profile_grid_and_progress():
    seen = []
    reports = profile(spring_counts=(1000, 3000), integrators=("euler", "verlet"), mode="serial",
                      progress=seen.append)
    assert [(r.spring_count, r.integrator) for r in reports] == [
        (block_springs(block_cells(1000)), "euler"), (block_springs(block_cells(1000)), "verlet"),
        (block_springs(block_cells(3000)), "euler"), (block_springs(block_cells(3000)), "verlet")]
    assert len(seen) == 4
    table = profile_table(reports)
    assert "springs/s" in table and "device:" in table
