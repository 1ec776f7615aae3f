"""GPU engine vs the reference's golden values (tests/golden/golden.json,
produced by the reference itself) on every node kind, the chi-squared path,
cached norms, counters, full fits, and the reference's error semantics.

Tolerances (BASELINE.json north_star): metric at fixed parameters <= 1e-12
relative; fitted parameters and uncertainties <= 1e-6 relative (scaled by
max(|p|, sigma_p) for parameters that converge near zero).
"""
import json
import math
import os
import sys

import numpy as np
import pytest

import oracle
from paper_1311_1753_b200 import parfit as pf

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from cases import CASES, FIT_CASES  # noqa: E402

with open(os.path.join(HERE, "golden", "golden.json")) as fh:
    GOLDEN = json.load(fh)["cases"]
REL = 1e-12


def fh(s):
    return float.fromhex(s)


@pytest.mark.parametrize("name", sorted(CASES))
def test_metric_norms_counters_vs_reference(name):
    g = GOLDEN[name]
    pdf, ds, grid, _ = CASES[name](pf)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    assert [p.name for p in bm.registry().parameters()] == g["param_names"]
    metric = pf.MetricKind(g["metric"])
    nodes = pf.GraphDesc(pdf, ds.observables()).preorder()
    for pt in g["points"]:
        p = [fh(v) for v in pt["params"]]
        got, want = bm.eval_metric(p, metric), fh(pt["value"])
        assert abs(got - want) <= REL * abs(want), (name, p, got, want)
        for node, n, v in zip(nodes, pt["norms"], pt["norm_valid"]):
            if v:
                assert abs(node.cached_norm() - fh(n)) <= REL * abs(fh(n)), (name, node.name())
        assert bm.log_floor_count() == pt["floor_count"], name
        if name == "polynomial":  # clamps: every raw call of grid and events (pdf.hpp:313-316)
            assert nodes[0].clamp_count() == pt["clamp"][0]


@pytest.mark.parametrize("name", FIT_CASES)
def test_fit_vs_reference(name):
    """parfit::fit (fit.hpp:498-581) driven by the GPU metric; batched FD probes."""
    g = GOLDEN[name]["fit"]
    pdf, ds, grid, _ = CASES[name](pf)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    metric = pf.MetricKind(GOLDEN[name]["metric"])
    r = pf.fit(bm, metric)
    assert r.status == pf.FitStatus(g["status"])
    assert r.uncertainties_available == g["uncertainties_available"]
    want_p = [fh(v) for v in g["params"]]
    want_u = [fh(v) for v in g["uncertainties"]]
    for got, want, sig in zip(r.params, want_p, want_u):
        assert abs(got - want) <= 1e-6 * max(abs(want), sig), (name, r.params, want_p)
    for got, want in zip(r.uncertainties, want_u):
        assert abs(got - want) <= 1e-6 * max(abs(want), 1e-300) or (want == 0 and got == 0), (name, r.uncertainties,
                                                                                              want_u)
    assert abs(r.metric_value - fh(g["metric_value"])) <= REL * abs(fh(g["metric_value"])) + 1e-9
    # written back into the Variables (fit.hpp:556)
    assert [p.value for p in bm.registry().parameters()] == r.params


def test_fit_sequential_probes_equal_batched():
    """batching the FD stencil changes no value: identical fits"""
    pdf, ds, grid, _ = CASES["listing1"](pf)
    bm = pf.BoundModel(pdf, ds)
    r1 = pf.fit(bm, cfg=pf.FitConfig(batch_probes=True))
    pdf, ds, grid, _ = CASES["listing1"](pf)
    bm = pf.BoundModel(pdf, ds)
    r2 = pf.fit(bm, cfg=pf.FitConfig(batch_probes=False))
    assert r1.params == r2.params and r1.uncertainties == r2.uncertainties
    assert r1.n_metric_calls == r2.n_metric_calls and r1.metric_value == r2.metric_value


def test_nelder_mead_agrees():
    """test_fit.cpp:253-269"""
    pdf, ds, grid, _ = CASES["listing1"](pf)
    qn = pf.fit(pf.BoundModel(pdf, ds))
    pdf, ds, grid, _ = CASES["listing1"](pf)
    nm = pf.fit(pf.BoundModel(pdf, ds), cfg=pf.FitConfig(minimizer=pf.MinimizerKind.NelderMead))
    assert qn.converged() and nm.converged()
    assert abs(qn.metric_value - nm.metric_value) <= 1e-4


def test_mapped_out_of_domain_raises_like_reference():
    """pdf.hpp:443-444: an event outside the mapped range throws from eval"""
    x = pf.new_observable("x", 0, 10)
    c1, c2 = pf.new_parameter("c1", 1, 0.1, 0.5, 5), pf.new_parameter("c2", 2, 0.1, 0.5, 5)
    pdf = pf.mapped_pdf("step", [0, 5, 10], [pf.polynomial_pdf("lo", x, [c1]), pf.polynomial_pdf("hi", x, [c2])])
    ds = pf.UnbinnedDataSet.from_columns([x], [2.0, 5.0, 7.0, 10.5, 3.0])
    with pytest.raises(pf.Error, match="out-of-domain"):
        pf.BoundModel(pdf, ds).eval_metric([1.0, 2.0])
    if oracle.Reference.available():
        with pytest.raises(oracle.OracleError, match="out-of-domain"):
            oracle.Reference(pdf, ds).eval([1.0, 2.0])


def test_nonfinite_reports_first_index():
    """engine.hpp:210-216: NaN data -> non-finite-metric with the first index"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -1, 0.1, -10, 10)
    vals = 10.0 * oracle.mt64_uniform(3, 100_000)
    vals[77_777] = math.nan
    vals[90_001] = math.nan
    ds = pf.UnbinnedDataSet.from_columns([x], vals)
    with pytest.raises(pf.Error, match="non-finite-metric: first offending event index 77777"):
        pf.BoundModel(pf.exp_pdf("e", x, a), ds).eval_metric([-1.0])
    if oracle.Reference.available():
        with pytest.raises(oracle.OracleError, match="first offending event index 77777"):
            oracle.Reference(pf.exp_pdf("e2", x, a), ds).eval([-1.0])


def test_degenerate_norm_is_penalty_and_fit_survives():
    """test_fit.cpp:288-301: zero integral -> 1e300; the fit reports, not throws"""
    x = pf.new_observable("x", 0, 10)
    m = pf.new_parameter("m", 100, 0.5, 50, 200)
    s = pf.new_parameter("s", 0.5, 0.1, 0.01, 5)
    ds = pf.UnbinnedDataSet.from_columns([x], [5.0])
    bm = pf.BoundModel(pf.gaussian_pdf("far", x, m, s), ds)
    assert bm.eval_metric([100.0, 0.5]) == pf.kPenaltyValue
    r = pf.fit(bm)
    assert r.status != pf.FitStatus.Failed and r.metric_value == pf.kPenaltyValue


def test_size_mismatch_and_metric_mismatch():
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -1, 0.1, -10, 10)
    bm = pf.BoundModel(pf.exp_pdf("e", x, a), pf.UnbinnedDataSet.from_columns([x], [1.0, 2.0]))
    with pytest.raises(pf.Error, match="size-mismatch"):
        bm.eval_metric([-1.0, 2.0])
    with pytest.raises(pf.Error, match="metric-mismatch"):
        bm.eval_metric([-1.0], pf.MetricKind.ChiSquared)


def test_fixed_parameters_hold():
    """test_fit.cpp:196-229"""
    x = pf.new_observable("x", -5, 5)
    mean = pf.new_parameter("mean", 0.3, 0.5, -4, 4)
    sigma = pf.new_parameter("sigma", 1.0, 0.5, 0.2, 4)
    sigma.fixed = True
    from cases import box_muller
    bm = pf.BoundModel(pf.gaussian_pdf("g", x, mean, sigma), pf.UnbinnedDataSet.from_columns([x], box_muller(31, 2000)))
    r = pf.fit(bm)
    assert r.converged() and r.params[1] == 1.0 and r.uncertainties[1] == 0.0 and r.uncertainties[0] > 0
    mean2 = pf.new_parameter("mean", 0.3, 0.5, -4, 4)
    mean2.fixed = True
    bm2 = pf.BoundModel(pf.gaussian_pdf("g2", x, mean2, sigma), pf.UnbinnedDataSet.from_columns([x], [0.1]))
    with pytest.raises(pf.Error, match="no-parameters"):
        pf.fit(bm2)


def test_report_keys():
    """test_fit.cpp:303-314"""
    pdf, ds, grid, _ = CASES["listing1"](pf)
    rep = pf.fit(pf.BoundModel(pdf, ds)).to_report()
    for key in ("status ", "metric_value ", "metric_calls ", "wall_time_s ", "grad_max_norm ",
                "uncertainties ", "param alpha "):
        assert key in rep


def test_shards_in_one_process_match_single_device():
    """single-process multi-shard path (one device, shard_count > 1 via two
    models): the exact accumulators combine to the single-device value"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.6, 0.1, -5, 5)
    m = pf.new_parameter("m", 5, 0.1, 0, 10)
    s = pf.new_parameter("s", 1, 0.1, 0.1, 5)
    f = pf.new_parameter("f", 0.4, 0.01, 0, 1)
    pdf = pf.add_pdf("mix", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s)], [f])
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(31, 1_000_000))
    p = [0.4, -0.6, 5, 1]
    whole = pf.BoundModel(pdf, ds).eval_metric(p)
    for G in (2, 4, 8):
        parts = []
        for r in range(G):
            fx, pen = pf.BoundModel(pdf, ds, shard_index=r, shard_count=G).eval_partial(p)
            assert not pen
            parts.append(fx)
        assert pf.combine_partials(parts) == whole
