"""The C oracle (oracle/pf_oracle.c) pinned against the reference.

Golden values in tests/golden/golden.json come from the reference's own
BoundModel / fit compiled from /root/reference (make_golden.py); the oracle
restatement must reproduce them (it follows the same expression order, libm
and long-double accumulation).  CPU only.
"""
import json
import math
import os
import sys

import numpy as np
import pytest

import oracle
from paper_1311_1753_b200 import parfit as pf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from cases import CASES  # noqa: E402

with open(os.path.join(HERE, "golden", "golden.json")) as fh:
    GOLDEN = json.load(fh)["cases"]


def fh(s):
    return float.fromhex(s)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_golden(name):
    g = GOLDEN[name]
    pdf, ds, grid, _ = CASES[name](pf)
    o = oracle.Oracle(pdf, ds, grid)
    assert o.param_names() == g["param_names"]
    for pt in g["points"]:
        p = [fh(v) for v in pt["params"]]
        got = o.eval(p, g["metric"])
        want = fh(pt["value"])
        assert got == want or abs(got - want) <= 1e-15 * abs(want), (name, p, got, want)
        norms, errs, valid = o.norms()
        for i, (n, v) in enumerate(zip(pt["norms"], pt["norm_valid"])):
            if v:
                assert abs(norms[i] - fh(n)) <= 1e-15 * abs(fh(n)), (name, i)
        assert o.floor_count() == pt["floor_count"]


def test_golden_acceptance_value():
    """acceptance.cpp:346 prints 3218448.5501374062"""
    assert fh(GOLDEN["mixture_acceptance"]["points"][0]["value"]) == 3218448.5501374062


def test_reduce_basics():
    """test_engine.cpp:17-34"""
    assert oracle.reduce([]) == 0.0
    assert oracle.reduce([3.25]) == 3.25
    assert oracle.reduce([1, 2, 3, 4]) == 10.0
    u = oracle.mt64_uniform(123, 1_000_000) - 0.5
    r1, r2 = oracle.reduce(u), oracle.reduce(u)
    assert r1 == r2
    assert abs(r1 - math.fsum(u)) <= 1e-12 * abs(math.fsum(u))


def test_three_event_exponential():
    """test_engine.cpp:82-97 against the antiderivative"""
    x = pf.new_observable("x", 0, 21.49)
    alpha = pf.new_parameter("alpha", -2, 0.1, -10, 10)
    ds = pf.UnbinnedDataSet.from_columns([x], [3.0, 5.0, 1.0])
    nll = oracle.Oracle(pf.exp_pdf("e", x, alpha), ds).eval([-2.0])
    norm = (1.0 - math.exp(-2.0 * 21.49)) / 2.0
    assert nll == pytest.approx(-(-2.0 * 9) + 3 * math.log(norm), rel=1e-9)


def test_floor_and_penalty():
    """test_engine.cpp:150-186"""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 0, 0.1, -5, 5)
    c1 = pf.new_parameter("c1", 1, 0.1, -5, 5)
    o = oracle.Oracle(pf.polynomial_pdf("ramp", x, [c0, c1]), pf.UnbinnedDataSet.from_columns([x], [0.0, 5.0]))
    assert math.isfinite(o.eval([0.0, 1.0]))
    assert o.floor_count() == 1
    a = pf.new_parameter("a", -2, 0.1, -10, 10)
    m = pf.new_parameter("m", 5, 0.1, 0, 10)
    s = pf.new_parameter("s", 1, 0.1, 0.1, 5)
    f1 = pf.new_parameter("f1", 0.8, 0.01, 0, 1)
    f2 = pf.new_parameter("f2", 0.8, 0.01, 0, 1)
    pdf = pf.add_pdf("mix", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s),
                             pf.gaussian_pdf("g2", x, m, s)], [f1, f2])
    o = oracle.Oracle(pdf, pf.UnbinnedDataSet.from_columns([x], [5.0]))
    assert o.eval([0.8, 0.8, -2, 5, 1]) == 1e300


def test_argus_restatement():
    """ArgusPdf has no reference kernel (parity unpinned): check the oracle's
    restatement against its closed form x (1 - r^2)^p exp(c (1 - r^2))."""
    y = pf.new_observable("y", 5.20, 5.29)
    m0 = pf.new_parameter("m0", 5.29, 0.001, 5.0, 6.0)
    c = pf.new_parameter("c", -20.0, 0.1, -100, 0)
    p = pf.new_parameter("p", 0.5, 0.1, 0, 5)
    pdf = pf.argus_pdf("argus", y, m0, c, p)
    pts = np.array([[5.21, 5.25, 5.285, 5.29]])
    o = oracle.Oracle(pdf, pf.UnbinnedDataSet.from_columns([y], pts[0]))
    dens = o.density([5.29, -20.0, 0.5], pts)
    raw = [v * (1 - (v / 5.29) ** 2) ** 0.5 * math.exp(-20 * (1 - (v / 5.29) ** 2)) if v < 5.29 else 0.0
           for v in pts[0]]
    norm = dens[0] and raw[0] / dens[0]
    for d, r in zip(dens, raw):
        assert d == pytest.approx(r / norm, rel=1e-12, abs=1e-300)


def test_mt64_matches_std():
    """std::mt19937_64 default seed 5489: 10000th output is 9981545732273789042"""
    u = oracle.mt64_uniform(5489, 10000)
    assert int(u[-1] * 2 ** 53) == 9981545732273789042 >> 11


def test_dalitz_restatement_vs_numpy():
    """DalitzPlotPdf has no reference code (parity unpinned): the C oracle's
    amplitude is checked against an independent numpy implementation of the
    same formulas (workloads.dalitz_amplitude2): density / |A|^2 must be the
    constant 1/norm at every point of the plot, and 0 outside."""
    import numpy as np
    from paper_1311_1753_b200.workloads import WORKLOADS, dalitz_amplitude2
    W = WORKLOADS["C5TI"]
    obs, pdf = W.build(pf)
    pts = W.columns(2000, seed=3)
    ds = pf.UnbinnedDataSet.from_columns(obs, pts)
    o = oracle.Oracle(pdf, ds, 64)
    names = o.param_names()
    p = [W.truth[n] for n in names]
    dens = o.density(p, pts)
    res = [(m, w, re, im, ch, sp) for _, ch, sp, m, w, re, im in W.res]
    ref = dalitz_amplitude2(pts[0], pts[1], W.M, W.ms, W.R, res)
    ratio = dens / ref
    assert np.all(ref > 0)
    assert np.max(np.abs(ratio / ratio[0] - 1.0)) < 1e-12
    (a12, b12), (a13, b13) = W.box()
    corner = np.array([[b12 - 1e-6], [b13 - 1e-6]])  # far outside the plot
    assert o.density(p, corner)[0] == 0.0


def test_generate_restatement_matches_reference_samples():
    """the test-side restatement of generate_events (ToyRng stream + the C
    oracle's densities, tests/golden/gen_cases.py) reproduces the reference's
    samples bit for bit (tests/golden/generate.json, made by oracle/_ref)"""
    import hashlib
    import json
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    from gen_cases import CASES, restated_generate
    golden = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "generate.json")))
    for name in ("exp_seed42", "uniform", "gauss", "bw", "mixture", "composite_mapped", "criterion2"):
        pdf, obs, n, seed, grid = CASES[name](pf)
        cols = restated_generate(pf, pdf, obs, n, seed, grid)
        assert hashlib.sha256(np.ascontiguousarray(cols).tobytes()).hexdigest() == golden[name]["sha256"], name


def _tddp_case(n=2000, seed=3):
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C5"]
    obs, pdf = W.build(pf)
    pts = W.columns(n, seed=seed)
    return W, obs, pdf, pts


def test_tddp_restatement_vs_numpy():
    """TddpPdf has no reference code (parity unpinned): the C oracle's
    expanded density is checked against an independent numpy evaluation of
    the complex form |A g+ + Abar g-|^2 (workloads.tddp_density): density /
    numpy must be the constant 1/norm, for physical and exaggerated mixing"""
    import numpy as np
    from paper_1311_1753_b200.workloads import tddp_density
    W, obs, pdf, pts = _tddp_case()
    ds = pf.UnbinnedDataSet.from_columns(obs, pts)
    o = oracle.Oracle(pdf, ds, 16)
    names = o.param_names()
    res = [(m, w, re, im, ch, sp) for _, ch, sp, m, w, re, im in W.res]
    for tau, x, y in ((W.tau, W.x_mix, W.y_mix), (0.41, 0.15, -0.12), (0.35, -0.08, 0.19)):
        p = [W.truth[nm] for nm in names]
        p[names.index("tau")], p[names.index("x")], p[names.index("y")] = tau, x, y
        dens = o.density(p, pts)
        ref = tddp_density(pts[0], pts[1], pts[2], W.M, W.ms, W.R, res, tau, x, y)
        assert np.all(ref > 0)
        ratio = dens / ref
        assert np.max(np.abs(ratio / ratio[0] - 1.0)) < 1e-12, (tau, x, y)


def test_tddp_separable_norm_is_the_3d_midpoint_sum():
    """the oracle (and the GPU) normalise a TddpPdf by the separable form of
    the 3-D midpoint sum; at a small grid it equals the brute-force walk over
    all n^3 (s12, s13, t) points (midpoint_sum, pdf.hpp:148-176) to rounding"""
    W, obs, pdf, pts = _tddp_case(500)
    ds = pf.UnbinnedDataSet.from_columns(obs, pts)
    names = oracle.Oracle(pdf, ds, 12).param_names()
    p = [W.truth[nm] for nm in names]
    p[names.index("x")], p[names.index("y")] = 0.15, -0.12
    sep = oracle.Oracle(pdf, ds, 12)
    a = sep.eval(p)
    os.environ["PO_TDDP_BRUTE"] = "1"
    try:
        brute = oracle.Oracle(pdf, ds, 12)
        b = brute.eval(p)
    finally:
        del os.environ["PO_TDDP_BRUTE"]
    assert abs(a - b) <= 1e-13 * abs(b)
    assert abs(sep.norms()[0][0] - brute.norms()[0][0]) <= 1e-13 * abs(brute.norms()[0][0])
