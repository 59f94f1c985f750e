"""Serving strategies (paper's sequential / concurrent / hybrid baselines,
PAPER.md:391-399, and the reference bench strategies,
pkg/src/modelmerge/bench.py:102-199): host logic on CPU, one short run of
every strategy on the GPU."""
import pytest

from paper_2009_13062_b200 import serving as S


def test_partition_balanced_contiguous():
    assert S.partition(8, 1) == [list(range(8))]
    assert S.partition(8, 8) == [[i] for i in range(8)]
    parts = S.partition(32, 5)
    assert [len(p) for p in parts] == [7, 7, 6, 6, 6]
    assert sum(parts, []) == list(range(32))


@pytest.mark.parametrize("bad", [(0, 1), (4, 0), (4, 5)])
def test_partition_rejects(bad):
    with pytest.raises(ValueError):
        S.partition(*bad)


def test_resolve():
    assert S.resolve("sequential", 32) == ("sequential", 1)
    assert S.resolve("concurrent", 32) == ("concurrent", 32)
    assert S.resolve("merged", 32) == ("merged", 1)
    assert S.resolve("hybrid:4", 32) == ("hybrid", 4)
    assert S.resolve("hybrid", 32, processes=8) == ("hybrid", 8)
    for bad in ("threaded", "hybrid", "hybrid:0", "hybrid:33", "merged:2"):
        with pytest.raises(ValueError):
            S.resolve(bad, 32)


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["sequential", "concurrent", "hybrid:2", "merged"])
def test_serving_strategy_runs(strategy):
    r = S.run_serving("bert-2l", strategy, 4, batch=1, rounds=3, warmup=1)
    assert r.error is None, r.error
    assert r.inferences_per_s > 0 and r.wall_s > 0
    assert sum(r.models_per_process) == 4
    assert len(r.worker_allocated_bytes) == r.processes
    assert all(b > 0 for b in r.worker_allocated_bytes)
    assert r.kernel_launches_per_round > 0
