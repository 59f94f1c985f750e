"""bench.py host logic on CPU: weak / strong instance sharding, BASELINE
config resolution, and the bounded reference-CPU sample (one job)."""

import argparse

import pytest

import bench


def _ns(**kw):
    base = dict(model="bert-base", instances=32, batch=8, dtype="bf16", config="C5",
                scaling="weak")
    base.update(kw)
    return argparse.Namespace(**base)


def test_weak_and_strong_shards_cover_the_instances():
    for world in (1, 2, 4, 8):
        weak = [bench.shard_for(_ns(), world, r) for r in range(world)]
        assert [i for s in weak for i in s] == list(range(32 * world))
        assert all(len(s) == 32 for s in weak)
        strong = [bench.shard_for(_ns(instances=256, scaling="strong"), world, r)
                  for r in range(world)]
        assert [i for s in strong for i in s] == list(range(256))
        assert all(len(s) == 256 // world for s in strong)


def test_default_is_the_c5_shard(monkeypatch, capsys):
    seen = {}
    monkeypatch.setattr(bench, "run_ours", lambda a: seen.setdefault("args", a) and None)
    bench.main([])
    a = seen["args"]
    assert (a.model, a.instances, a.batch, a.dtype, a.config) == ("bert-base", 32, 8, "bf16",
                                                                 "C5")
    bench.main(["--config", "C1"])
    assert seen["args"].dtype == "bf16"  # first call's args kept by setdefault
    seen.clear()
    bench.main(["--config", "C1"])
    assert (seen["args"].model, seen["args"].instances, seen["args"].dtype) == ("resnet50", 2,
                                                                               "f32")
    seen.clear()
    bench.main(["--config", "C2", "--instances", "4"])
    assert seen["args"].config is None  # not the named config any more


def test_reference_sample_is_one_layer_of_one_sequence():
    s = bench.ReferenceSampler(_ns(instances=1), [0])
    items, secs = s.step(1)
    assert items == pytest.approx(1 / 12) and secs > 0
    assert "1 of 12 encoder layers" in s.unit
