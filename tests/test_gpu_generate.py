"""GPU toy generation (generate_events, generate.hpp:33-86) against the
reference.

  * every case of tests/golden/gen_cases.py (the reference's own
    generate_events calls): sha256 of the GPU sample == the reference's
    (tests/golden/generate.json, made by oracle/_ref), plus the first/last
    events and the observables' final values;
  * when oracle/_ref is present: a 1e6-event sample compared event by event;
    envelope-failure and zero-integral raised like the reference;
  * PDFs the reference lacks (ArgusPdf, DalitzPlotPdf): against a restatement
    of generate_events built from ToyRng draws (oracle.mt64_uniform) and the
    C oracle's densities;
  * the reference's statistical checks (test_generate.cpp) on GPU samples.
"""
import hashlib
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
from gen_cases import CASES, restated_generate  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = json.load(open(os.path.join(HERE, "golden", "generate.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_sample_is_the_reference_sample(name):
    pdf, obs, n, seed, grid = CASES[name](pf)
    ds = pf.generate_events(pdf, obs, n, seed, pf.GridSpec(grid))
    cols = ds.columns()
    want = GOLDEN[name]
    assert cols.shape == (len(obs), want["n"])
    assert [repr(float(v)) for v in cols[:, 0]] == want["first"]
    assert [repr(float(v)) for v in cols[:, -1]] == want["last"]
    assert hashlib.sha256(np.ascontiguousarray(cols).tobytes()).hexdigest() == want["sha256"]
    # the reference leaves each box observable at the last accepted event
    assert [o.value for o in obs] == [float(v) for v in want["last"]]


def test_million_events_equal_reference():
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built")
    pdf, obs, _, _, grid = CASES["mixture"](pf)
    got = pf.generate_events(pdf, obs, 1_000_000, 11).columns()
    want = oracle.ref_generate(pdf, obs, 1_000_000, 11, grid)
    assert np.array_equal(got, want)


def test_same_seed_same_sample_other_seed_differs():
    """test_generate.cpp:37-47"""
    pdf, obs, n, seed, _ = CASES["exp_seed42"](pf)
    a = pf.generate_events(pdf, obs, n, seed).columns()
    b = pf.generate_events(pdf, obs, n, seed).columns()
    c = pf.generate_events(pdf, obs, n, seed + 1).columns()
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


def _narrow():
    x = pf.new_observable("x", 0, 10)
    return pf.gaussian_pdf("g", x, pf.new_parameter("m", 5.0031, 0.1, 0, 10),
                           pf.new_parameter("s", 0.0005, 0.1, 1e-6, 5)), [x]


def test_envelope_failure_like_reference():
    """a peak narrower than a grid cell exceeds the 1.1 x grid-maximum
    envelope (generate.hpp:72-76)"""
    pdf, obs = _narrow()
    with pytest.raises(pf.Error) as got:
        pf.generate_events(pdf, obs, 1000, 1)
    assert got.value.code == "envelope-failure"
    if oracle.Reference.available():
        with pytest.raises(oracle.OracleError) as want:
            oracle.ref_generate(pdf, obs, 1000, 1)
        assert str(want.value) == str(got.value)


def test_zero_integral_like_reference():
    x = pf.new_observable("x", 0, 10)
    pdf = pf.gaussian_pdf("far", x, pf.new_parameter("m", 1e4, 0.1, -1e5, 1e5),
                          pf.new_parameter("s", 1.0, 0.1, 0.1, 5))
    with pytest.raises(pf.Error) as got:
        pf.generate_events(pdf, [x], 100, 1)
    assert got.value.code == "zero-integral"
    if oracle.Reference.available():
        with pytest.raises(oracle.OracleError) as want:
            oracle.ref_generate(pdf, [x], 100, 1)
        assert want.value.code == "zero-integral"


def test_bad_arity():
    """test_generate.cpp:141-146"""
    pdf, obs, _, _, _ = CASES["exp_seed42"](pf)
    with pytest.raises(pf.Error, match="n_events"):
        pf.generate_events(pdf, obs, 0, 1)


def test_argus_sample_vs_restatement():
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C3"]
    obs, pdf = W.build(pf)
    got = pf.generate_events(pdf, obs, 3000, 17, pf.GridSpec(256)).columns()
    want = restated_generate(pf, pdf, obs, 3000, 17, 256)
    assert np.array_equal(got, want)


def test_dalitz_sample_vs_restatement():
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C5TI"]
    obs, pdf = W.build(pf)
    got = pf.generate_events(pdf, obs, 2000, 23, pf.GridSpec(256)).columns()
    want = restated_generate(pf, pdf, obs, 2000, 23, 256)
    assert np.array_equal(got, want)


def test_tddp_sample_vs_restatement():
    """the time-dependent Dalitz model (3-D box: m12^2, m13^2, t; 4 ToyRng
    words per candidate) through the same generator: bit for bit the
    restatement over the C oracle's densities, at exaggerated mixing"""
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C5"]
    obs, pdf = W.build(pf)
    for v in pf.GraphDesc(pdf, obs).vars:
        if v.name in ("x", "y"):
            v.value = 0.15 if v.name == "x" else -0.12
    # grid 128: the envelope (1.1 x the midpoint-grid maximum, generate.hpp)
    # must cover the t = 0 edge of e^-t/tau (a coarser grid raises
    # envelope-failure, as the reference would)
    got = pf.generate_events(pdf, obs, 2000, 29, pf.GridSpec(128)).columns()
    want = restated_generate(pf, pdf, obs, 2000, 29, 128)
    assert np.array_equal(got, want)


# ---- the reference's statistical checks (test_generate.cpp), on GPU samples --

def test_uniform_density_gives_uniform_sample():
    """test_generate.cpp:50-67"""
    pdf, obs, n, seed, _ = CASES["uniform"](pf)
    x = pf.generate_events(pdf, obs, n, seed).columns()[0]
    sd = 6.0 / math.sqrt(12.0 * n)
    assert abs(x.mean() - 5.0) < 5 * sd
    assert x.min() >= 2.0 and x.max() <= 8.0


def test_exponential_cdf_deciles():
    """test_generate.cpp:69-87"""
    pdf, obs, n, seed, _ = CASES["exp_cdf"](pf)
    xs = np.sort(pf.generate_events(pdf, obs, n, seed).columns()[0])
    for q in (1.0, 2.0, 3.0, 5.0, 8.0):
        f = (math.exp(-0.7 * q) - 1.0) / (math.exp(-0.7 * 10.0) - 1.0)
        emp = np.searchsorted(xs, q, side="right") / n
        assert abs(emp - f) < 5 * math.sqrt(f * (1 - f) / n)


def test_gaussian_moments():
    """test_generate.cpp:89-104"""
    pdf, obs, n, seed, _ = CASES["gauss"](pf)
    x = pf.generate_events(pdf, obs, n, seed).columns()[0]
    assert abs(x.mean() - 1.2) < 5 * 0.8 / math.sqrt(n)
    assert x.var(ddof=1) == pytest.approx(0.64, rel=0.05)


def test_product_factorizes():
    """test_generate.cpp:106-126"""
    pdf, obs, n, seed, _ = CASES["prod2d"](pf)
    cols = pf.generate_events(pdf, obs, n, seed).columns()

    def expect(a, u):
        return 1.0 / -a - u / (math.exp(-a * u) - 1.0)

    assert cols[0].mean() == pytest.approx(expect(-2.4, 5.0), rel=0.03)
    assert cols[1].mean() == pytest.approx(expect(-1.1, 5.0), rel=0.03)


def test_generated_sample_closes_the_loop_with_the_fitter():
    """test_generate.cpp:128-139"""
    pdf, obs, n, seed, _ = CASES["closure"](pf)
    ds = pf.generate_events(pdf, obs, n, seed)
    afit = pf.new_parameter("a", -0.3, 0.2, -5, -0.05)
    bm = pf.BoundModel(pf.exp_pdf("fit", obs[0], afit), ds)
    res = pf.fit(bm, pf.MetricKind.NegLogLikelihood)
    assert res.converged() and res.uncertainties_available
    assert abs(res.params[0] + 0.7) < 5 * res.uncertainties[0]


def test_ten_million_events_mixture_fraction():
    """C2-sized sample (1e7): size-independent properties — every event in
    the box, the Gaussian-window population matches the truth mixture"""
    pdf, obs, _, _, _ = CASES["mixture"](pf)
    ds = pf.generate_events(pdf, obs, 10_000_000, 11)
    x = ds.columns()[0]
    assert x.size == 10_000_000 and x.min() >= 0.0 and x.max() < 10.0
    # P(x < 2): 0.3 * Gauss(5, 0.8) part (negligible) + 0.7 * truncated Exp(-0.6)
    f_exp = 0.7 * (math.exp(-0.6 * 2.0) - 1.0) / (math.exp(-0.6 * 10.0) - 1.0)
    g = 0.3 * 0.5 * (math.erfc(3.0 / (0.8 * math.sqrt(2))) -
                     math.erfc(5.0 / (0.8 * math.sqrt(2)))) / (1 - 2 * 0.5 * math.erfc(5.0 / (0.8 * math.sqrt(2))))
    p = f_exp + g
    emp = float(np.mean(x < 2.0))
    assert abs(emp - p) < 5 * math.sqrt(p * (1 - p) / x.size)


def test_sequential_stream_path_gives_the_same_sample(monkeypatch):
    """PFB200_MT_SEQUENTIAL forces the one-CTA stream (the path for candidates
    whose word count does not divide a twist): same sample as the jump-ahead
    draw and as the reference"""
    pdf, obs, n, seed, grid = CASES["prod2d"](pf)
    jumped = pf.generate_events(pdf, obs, n, seed, pf.GridSpec(grid)).columns()
    monkeypatch.setenv("PFB200_MT_SEQUENTIAL", "1")
    seq = pf.generate_events(pdf, obs, n, seed, pf.GridSpec(grid)).columns()
    assert np.array_equal(jumped, seq)
    assert hashlib.sha256(np.ascontiguousarray(seq).tobytes()).hexdigest() == GOLDEN["prod2d"]["sha256"]


def test_four_dimensional_sample_vs_restatement():
    """4 observables: 5 words per candidate (does not divide 312), so the
    sequential stream; checked against the oracle restatement"""
    obs = [pf.new_observable(f"x{i}", 0, 5) for i in range(4)]
    pars = [pf.new_parameter(f"a{i}", -0.1 + 0.02 * i, 0.1, -5, 5) for i in range(4)]  # gentle slopes:
    pdf = pf.prod_pdf("p4", [pf.exp_pdf(f"e{i}", obs[i], pars[i]) for i in range(4)])  # the 16^4 grid's
    got = pf.generate_events(pdf, obs, 3000, 41, pf.GridSpec(16)).columns()  # max stays inside the envelope
    want = restated_generate(pf, pdf, obs, 3000, 41, 16)
    assert np.array_equal(got, want)
