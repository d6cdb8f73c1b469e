"""The reference's benchmark protocols on the GPU (mirrors pkg/tests/test_bench.py).
Report plumbing runs on CPU; the runs need the GPU."""

from __future__ import annotations

import dataclasses
import io
import json

import numpy as np
import pytest

from paper_2603_15486_b200 import analytic_fpr
from paper_2603_15486_b200.bench_harness import (BenchReport, RunSpec, emit_report, gen_keys, read_reports,
                                                 run_eviction_study, run_fpr_sweep, run_throughput)

SMALL = dict(bucket_count=1 << 8, repetitions=2, warmup=1)


def _rep(**kw):
    base = dict(op="query_pos", policy="xor", eviction="dfs", fingerprint_bits=16, bucket_slots=16,
                bucket_count=4, memory_bytes=512, load_factor=0.5, workers=1, seed=0, repetitions=1,
                warmup=0, n_keys=10, wall_time=0.25, throughput=40.0, empirical_fpr=None,
                analytic_fpr=1e-4, insert_failures=0, eviction_p90=None, eviction_p95=None,
                eviction_p99=None)
    base.update(kw)
    return BenchReport(**base)


def test_runspec_validation():
    RunSpec(bucket_count=16)
    for bad in [dict(op="mutate"), dict(load_factor=1.5), dict(workers=0), dict(repetitions=0),
                dict(warmup=-1), dict(mode="fast")]:
        with pytest.raises(ValueError):
            RunSpec(bucket_count=16, **bad)


def test_gen_keys_ranges_are_disjoint_and_seeded():
    pos, neg = gen_keys(50_000, seed=1), gen_keys(50_000, seed=1, negative=True)
    assert int(pos.max()) < 1 << 32 and int(neg.min()) >= 1 << 32
    assert np.array_equal(pos, gen_keys(50_000, seed=1))
    assert not np.array_equal(pos, gen_keys(50_000, seed=2))


def test_report_round_trips(tmp_path):
    reps = [_rep(), _rep(op="insert", eviction_p90=1, eviction_p95=2, eviction_p99=3, empirical_fpr=None),
            _rep(op="query_neg", empirical_fpr=1.5e-4)]
    for fmt, name in (("csv", "r.csv"), ("json", "r.json")):
        path = tmp_path / name
        emit_report(reps, fmt, path)
        assert read_reports(path) == reps
    buf = io.StringIO()
    emit_report([_rep()], "csv", buf)
    buf.seek(0)
    assert read_reports(buf, "csv") == [_rep()]
    empty = tmp_path / "e.csv"
    emit_report([], "csv", empty)
    assert empty.read_text().strip().startswith("op,policy,eviction,") and read_reports(empty) == []
    with pytest.raises(ValueError):
        emit_report([], "xml", io.StringIO())
    bad = tmp_path / "no" / "such" / "x.csv"
    with pytest.raises(OSError, match=str(bad)):
        emit_report([], "csv", bad)
    path = tmp_path / "n.json"
    emit_report([_rep()] * 3, "json", path)
    assert len(json.load(open(path))) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("op", ["insert", "query_pos", "query_neg", "delete"])
def test_run_throughput_all_ops(op):
    rep = run_throughput(RunSpec(op=op, **SMALL))
    assert rep.op == op and rep.throughput > 0 and rep.wall_time > 0
    assert rep.n_keys == int(0.95 * (1 << 8) * 16) and rep.insert_failures == 0
    if op == "query_neg":
        assert 0.0 <= rep.empirical_fpr <= 1.0
    else:
        assert rep.empirical_fpr is None
    if op == "insert":
        assert rep.eviction_p99 is not None and rep.eviction_p90 >= 0
    assert rep.analytic_fpr == pytest.approx(analytic_fpr(16, 16, 0.95))


@pytest.mark.gpu
def test_deterministic_mode_reports_repeat_apart_from_timing():
    def scrub(rep):
        return dataclasses.replace(rep, wall_time=0.0, throughput=0.0)

    spec = RunSpec(op="insert", seed=77, mode="deterministic", **SMALL)
    assert scrub(run_throughput(spec)) == scrub(run_throughput(spec))


@pytest.mark.gpu
def test_fpr_sweep_tracks_model():
    reports = run_fpr_sweep(RunSpec(bucket_count=1, seed=3), memory_bytes=[1 << 15, 1 << 16],
                            negative_queries=300_000)
    assert [r.bucket_count for r in reports] == [1 << 10, 1 << 11]
    for rep in reports:
        assert rep.op == "query_neg" and rep.insert_failures == 0
        assert 0.6 * rep.analytic_fpr < rep.empirical_fpr < 1.6 * rep.analytic_fpr
    (empty,) = run_fpr_sweep(RunSpec(bucket_count=1, load_factor=0.0), memory_bytes=[1 << 15],
                             negative_queries=50_000)
    assert empty.empirical_fpr == 0.0
    with pytest.raises(ValueError):
        run_fpr_sweep(RunSpec(bucket_count=1), memory_bytes=[8], negative_queries=10)


@pytest.mark.gpu
def test_eviction_study_direction():
    reports = run_eviction_study(RunSpec(bucket_count=1 << 8, seed=5), load_factors=[0.75, 0.95, 1.0])
    by = {(r.eviction, r.load_factor): r for r in reports}
    assert len(reports) == 6
    for s in ("dfs", "bfs"):
        assert by[(s, 0.75)].eviction_p99 <= 2
    for a in (0.95, 1.0):
        assert by[("bfs", a)].eviction_p99 <= by[("dfs", a)].eviction_p99
    assert by[("dfs", 1.0)].n_keys == (1 << 8) * 16 - (3 * (1 << 8) * 16) // 4
