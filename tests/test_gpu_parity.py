"""GPU parity: the CUDA path (through the C ABI) against the C oracle and the
compiled reference, on the reference tests' own inputs where they exist.

Tolerance (BASELINE.json north_star): NLL / chi2 at fixed parameters within
1e-12 relative of the CPU oracle.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1311_1753_b200 import parfit as pf

pytestmark = pytest.mark.gpu
REL = 1e-12


def close(a, b, rel=REL):
    return abs(a - b) <= rel * max(abs(a), abs(b))


def mixture(a=-0.6, m=5.0, s=1.0, f=0.4, lo=0.0, hi=10.0):
    x = pf.new_observable("x", lo, hi)
    av = pf.new_parameter("a", a, 0.1, -5, 5)
    mv = pf.new_parameter("m", m, 0.1, 0, 10)
    sv = pf.new_parameter("s", s, 0.1, 0.1, 5)
    fv = pf.new_parameter("f", f, 0.01, 0, 1)
    pdf = pf.add_pdf("mix", [pf.exp_pdf("e", x, av), pf.gaussian_pdf("g", x, mv, sv)], [fv])
    return x, pdf


def test_golden_acceptance_criterion5():
    """acceptance.cpp:305-348: 1e6 events, mt19937_64(31), x = 10 u;
    reference prints NLL 3218448.5501374062."""
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(31, 1_000_000))
    bm = pf.BoundModel(pdf, ds)
    assert [p.name for p in bm.registry().parameters()] == ["f", "a", "m", "s"]
    nll = bm.eval_metric(bm.registry().export_values())
    assert close(nll, 3218448.5501374062), f"{nll!r}"
    # node norms: e = 1.6625354130382941, g = 2.5066268375731329
    e, g = pdf.children()
    assert close(e.cached_norm(), 1.6625354130382941, 1e-14)
    assert close(g.cached_norm(), 2.5066268375731329, 1e-14)
    assert abs(pdf.cached_norm() - 1.0) < 1e-9


def test_three_event_exponential():
    """test_engine.cpp:82-97"""
    x = pf.new_observable("x", 0, 21.49)
    alpha = pf.new_parameter("alpha", -2, 0.1, -10, 10)
    ds = pf.UnbinnedDataSet(x)
    for v in (3.0, 5.0, 1.0):
        x.value = v
        ds.add_event()
    bm = pf.BoundModel(pf.exp_pdf("e", x, alpha), ds)
    nll = bm.eval_metric(bm.registry().export_values())
    norm = (1.0 - math.exp(-2.0 * 21.49)) / 2.0
    expect = -(-2.0 * (3 + 5 + 1)) + 3 * math.log(norm)
    assert abs(nll - expect) <= 1e-9 * abs(expect)
    o = oracle.Oracle(bm.pdf(), ds)
    assert close(nll, o.eval([-2.0]))


def test_empty_dataset_zero():
    """test_engine.cpp:52-59"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -2, 0.1, -10, 10)
    bm = pf.BoundModel(pf.exp_pdf("e", x, a), pf.UnbinnedDataSet(x))
    assert bm.eval_metric(bm.registry().export_values()) == 0.0


def test_uniform_single_event_log10():
    """test_engine.cpp:70-80"""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 1, 0.1, 0.5, 5)
    ds = pf.UnbinnedDataSet(x)
    x.value = 4.2
    ds.add_event()
    bm = pf.BoundModel(pf.polynomial_pdf("u", x, [c0]), ds)
    assert abs(bm.eval_metric(bm.registry().export_values()) - math.log(10.0)) <= 1e-10 * math.log(10)


def test_matched_bins_zero_chi2():
    """test_engine.cpp:99-109"""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 1, 0.1, 0.5, 5)
    b = pf.BinnedDataSet([x], [10])
    for i in range(10):
        b.fill([0.5 + i], 5.0)
    bm = pf.BoundModel(pf.polynomial_pdf("u", x, [c0]), b)
    assert abs(bm.eval_metric(bm.registry().export_values(), pf.MetricKind.ChiSquared)) <= 1e-15


def test_floor_counter():
    """test_engine.cpp:150-166"""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 0, 0.1, -5, 5)
    c1 = pf.new_parameter("c1", 1, 0.1, -5, 5)
    ds = pf.UnbinnedDataSet(x)
    for v in (0.0, 5.0):
        x.value = v
        ds.add_event()
    bm = pf.BoundModel(pf.polynomial_pdf("ramp", x, [c0, c1]), ds)
    nll = bm.eval_metric(bm.registry().export_values())
    assert math.isfinite(nll)
    assert bm.log_floor_count() == 1
    o = oracle.Oracle(bm.pdf(), ds)
    assert close(nll, o.eval(bm.registry().export_values()))


def test_penalty_for_fraction_sum():
    """test_engine.cpp:168-186"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -2, 0.1, -10, 10)
    m = pf.new_parameter("m", 5, 0.1, 0, 10)
    s = pf.new_parameter("s", 1, 0.1, 0.1, 5)
    f1 = pf.new_parameter("f1", 0.8, 0.01, 0, 1)
    f2 = pf.new_parameter("f2", 0.8, 0.01, 0, 1)
    pdf = pf.add_pdf("mix", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s),
                             pf.gaussian_pdf("g2", x, m, s)], [f1, f2])
    ds = pf.UnbinnedDataSet(x)
    x.value = 5
    ds.add_event()
    bm = pf.BoundModel(pdf, ds)
    assert bm.eval_metric(bm.registry().export_values()) == pf.kPenaltyValue


def test_metric_mismatch_raises():
    """test_engine.cpp:111-121"""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 1, 0.1, 0.5, 5)
    ds = pf.UnbinnedDataSet(x)
    x.value = 1
    ds.add_event()
    bm = pf.BoundModel(pf.polynomial_pdf("p", x, [c0]), ds)
    with pytest.raises(pf.Error, match="metric-mismatch"):
        bm.eval_metric(bm.registry().export_values(), pf.MetricKind.ChiSquared)


@pytest.mark.parametrize("n", [1, 255, 4096, 4097, 50_000, 1_000_003])
def test_mixture_vs_oracle_ragged(n):
    """backend-equivalence inputs (test_engine.cpp:123-148) at ragged sizes"""
    x, pdf = mixture(a=-0.7, m=5, s=1, f=0.5)
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(77, n))
    bm = pf.BoundModel(pdf, ds)
    o = oracle.Oracle(pdf, ds)
    rng = np.random.default_rng(n)
    for _ in range(4):
        p = [rng.uniform(0, 1), rng.uniform(-2, 0), rng.uniform(3, 7), rng.uniform(0.5, 2)]
        assert close(bm.eval_metric(p), o.eval(p))


def test_batch_is_bitwise_sequential():
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(5, 300_000))
    bm = pf.BoundModel(pdf, ds)
    rng = np.random.default_rng(3)
    P = np.array([[rng.uniform(0, 1), rng.uniform(-2, 0), rng.uniform(3, 7), rng.uniform(0.5, 2)]
                  for _ in range(40)])
    P[7, 0] = 1.5  # invalid fraction -> penalty in the batch too
    batch = bm.eval_metric_batch(P)
    seq = np.array([bm.eval_metric(p) for p in P])
    assert np.array_equal(batch, seq)
    assert batch[7] == pf.kPenaltyValue


def test_reference_matches_on_random_points():
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built")
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(9, 200_000))
    bm = pf.BoundModel(pdf, ds)
    r = oracle.Reference(pdf, ds)
    for p in ([0.4, -0.6, 5, 1], [0.1, -1.5, 4.2, 0.7], [0.9, -0.1, 6.1, 1.9]):
        assert close(bm.eval_metric(p), r.eval(p))


# --- BASELINE configurations C3 / C4 at oracle-sized inputs -----------------
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402


def test_c3_gauss_argus_product_vs_oracle():
    """C3 shape: ProdPdf(Gauss(x), Argus(y)), 2-D normalisation grid 1024 x 1024
    (the GPU factorises the separable grid; the oracle walks all 5.2M points).
    ArgusPdf has no reference code: parity is against the C restatement."""
    W = WORKLOADS["C3"]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(20_011, seed=5))
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
    o = oracle.Oracle(pdf, ds, W.grid)
    names = [p.name for p in bm.registry().parameters()]
    nodes = pf.GraphDesc(pdf, obs).preorder()
    for pt in (W.start, W.truth, dict(m=5.3, s=0.8, m0=5.29, c=-35.0, p=1.2)):
        p = [pt[n] for n in names]
        got, want = bm.eval_metric(p), o.eval(p)
        assert close(got, want), (pt, got, want)
        norms, _, valid = o.norms()
        assert valid[0] and close(nodes[0].cached_norm(), norms[0])


def test_c3_floor_at_the_argus_endpoint():
    """events at or beyond m0 have raw 0: floored at 1e-300 and counted"""
    W = WORKLOADS["C3"]
    obs, pdf = W.build(pf)
    cols = W.columns(5000, seed=6)
    cols[1, ::97] = W.truth["m0"]  # exactly at the endpoint
    ds = pf.UnbinnedDataSet.from_columns(obs, cols)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
    o = oracle.Oracle(pdf, ds, W.grid)
    p = [W.truth[n.name] for n in bm.registry().parameters()]
    assert close(bm.eval_metric(p), o.eval(p))
    assert bm.log_floor_count() == o.floor_count() > 0


def test_c4_binned_convolution_vs_reference():
    """C4 shape: BW (x) Gauss, Q = 1024, binned chi-squared (2000 bins here)"""
    W = WORKLOADS["C4"]
    obs, pdf = W.build(pf)
    ds = W.data(pf, obs, 2000, seed=3)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
    ref = oracle.Reference(pdf, ds, W.grid) if oracle.Reference.available() else oracle.Oracle(pdf, ds, W.grid)
    names = [p.name for p in bm.registry().parameters()]
    for pt in (W.start, W.truth, dict(m=2.9, w=0.35, rm=0.01, rs=0.06)):
        p = [pt[n] for n in names]
        got = bm.eval_metric(p, pf.MetricKind.ChiSquared)
        want = ref.eval(p, 1)
        assert close(got, want), (pt, got, want)


def _conv_model(alpha, sigma, lo=0.0, hi=10.0, q=1024, mean=0.0):
    x = pf.new_observable("x", lo, hi)
    a = pf.new_parameter("a", alpha, 0.1, -50, 50)
    m = pf.new_parameter("rm", mean, 0.01, -1, 1)
    s = pf.new_parameter("rs", sigma, 0.01, 0.01, 5)
    return x, pf.convolution_pdf("cv", pf.exp_pdf("e", x, a), pf.gaussian_pdf("res", x, m, s), q)


@pytest.mark.parametrize("alpha,sigma,hi", [(-10.0, 0.4, 10.0), (-20.0, 0.2, 10.0), (-10.0, 1.0, 20.0),
                                            (-5.0, 0.3, 10.0), (8.0, 0.5, 10.0)])
def test_conv_steep_model_vs_reference(alpha, sigma, hi):
    """ConvolutionPdf sums all Q quadrature points (pdf.hpp:476-493).  A
    lifetime (x) resolution model whose table spans e^100 needs far more than
    a fixed +-9 sigma window (2e-7 per event at alpha = -10,
    sigma = 0.4); the per-call window is chosen from the table's dynamic range
    and checked per event.  Unbinned NLL and binned chi2, vs oracle/_ref."""
    x, pdf = _conv_model(alpha, sigma, hi=hi)
    rng = np.random.default_rng(5)
    ds = pf.UnbinnedDataSet.from_columns([x], hi * rng.random(20011))
    bm = pf.BoundModel(pdf, ds)
    ref = oracle.Reference(pdf, ds) if oracle.Reference.available() else oracle.Oracle(pdf, ds)
    p = bm.registry().export_values()
    got, want = bm.eval_metric(p), ref.eval(p, 0)
    assert close(got, want), (got, want, abs(got - want) / abs(want))
    assert bm.log_floor_count() == ref.floor_count()
    # binned chi2 of the same model (C4's metric)
    b = pf.BinnedDataSet([x], [3001])
    xc = (np.arange(3001) + 0.5) * hi / 3001
    b.set_contents(np.floor(1e6 * np.exp(alpha * xc / 4) / np.exp(alpha * xc / 4).sum()) + 1)
    bb = pf.BoundModel(pdf, b)
    rb = oracle.Reference(pdf, b) if oracle.Reference.available() else oracle.Oracle(pdf, b)
    got, want = bb.eval_metric(p, pf.MetricKind.ChiSquared), rb.eval(p, 1)
    assert close(got, want), (got, want, abs(got - want) / abs(want))


def test_conv_resolution_mean_far_outside_the_quadrature_range():
    """x - m outside [L, U] by more than the window: every term is a far tail
    (the reference still sums them, e^-50-scale, not 0)"""
    x, pdf = _conv_model(-1.0, 0.05, hi=4.0, mean=0.9)
    rng = np.random.default_rng(6)
    ds = pf.UnbinnedDataSet.from_columns([x], 4.0 * rng.random(5003))
    bm = pf.BoundModel(pdf, ds)
    ref = oracle.Reference(pdf, ds) if oracle.Reference.available() else oracle.Oracle(pdf, ds)
    p = bm.registry().export_values()
    got, want = bm.eval_metric(p), ref.eval(p, 0)
    assert close(got, want), (got, want)
    assert bm.log_floor_count() == ref.floor_count()


@pytest.mark.parametrize("binned", [False, True])
def test_conv_polynomial_clamp_counter_per_raw_call(binned):
    """PolynomialPdf counts every raw() that clamps (pdf.hpp:313-316); inside a
    convolution the reference calls it for every (raw call, tau_j) pair, events
    and normalisation grid points alike (pdf.hpp:484-491)"""
    x = pf.new_observable("x", 0.0, 10.0)
    c0 = pf.new_parameter("c0", 1.0, 0.1, -5, 5)
    c1 = pf.new_parameter("c1", -0.15, 0.01, -5, 5)
    m = pf.new_parameter("rm", 0.0, 0.01, -1, 1)
    s = pf.new_parameter("rs", 0.3, 0.01, 0.01, 5)
    poly = pf.polynomial_pdf("p", x, [c0, c1])
    pdf = pf.convolution_pdf("cv", poly, pf.gaussian_pdf("res", x, m, s), 256)
    rng = np.random.default_rng(7)
    if binned:
        ds = pf.BinnedDataSet([x], [1000])
        ds.set_contents(np.floor(100 * rng.random(1000)) + 1)
    else:
        ds = pf.UnbinnedDataSet.from_columns([x], 6.0 * rng.random(4001))
    bm = pf.BoundModel(pdf, ds)
    ref = oracle.Reference(pdf, ds) if oracle.Reference.available() else oracle.Oracle(pdf, ds)
    metric = 1 if binned else 0
    for k in range(2):
        p = bm.registry().export_values()
        got, want = bm.eval_metric(p, pf.MetricKind(metric)), ref.eval(p, metric)
        assert close(got, want), (got, want)
        assert poly.clamp_count() == ref.clamp_count(1) > 0, (k, poly.clamp_count(), ref.clamp_count(1))


def _folded_poly_models():
    x = pf.new_observable("x", 0.0, 4.0)
    y = pf.new_observable("y", 0.0, 2.0)
    c0 = pf.new_parameter("c0", 1.0, 0.1, -5, 5)
    c1 = pf.new_parameter("c1", -0.4, 0.1, -5, 5)
    a = pf.new_parameter("a", -1.0, 0.1, -5, 5)
    b = pf.new_parameter("b", -0.5, 0.1, -5, 5)
    f = pf.new_parameter("f", 0.5, 0.01, 0, 1)
    g = pf.new_parameter("g", 0.3, 0.01, 0, 1)
    poly = pf.polynomial_pdf("p", x, [c0, c1])
    inner = pf.add_pdf("in", [poly, pf.exp_pdf("e", x, a)], [f])
    yield "folded-add", pf.add_pdf("out", [inner, pf.exp_pdf("e2", x, b)], [g]), [x]
    poly2 = pf.polynomial_pdf("p2", x, [c0, c1])
    yield "separable-product", pf.prod_pdf("pr", [poly2, pf.exp_pdf("ey", y, b)]), [x, y]


@pytest.mark.parametrize("case", ["folded-add", "separable-product"])
def test_polynomial_clamps_under_folded_normalisations(case):
    """the reference walks the grid of every normalised node, folded or not
    (pdf.hpp:148-176), so a polynomial's clamps count once per reference raw
    call on those grids too; this engine folds AddPdf / separable ProdPdf
    norms from the children's sums and scales the children's counts"""
    name, pdf, obs = [m for m in _folded_poly_models() if m[0] == case][0]
    rng = np.random.default_rng(9)
    ds = pf.UnbinnedDataSet.from_columns(obs, np.stack([o.lower + (o.upper - o.lower) * rng.random(3001)
                                                        for o in obs]))
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(64))
    ref = oracle.Reference(pdf, ds, 64) if oracle.Reference.available() else oracle.Oracle(pdf, ds, 64)
    nodes = pf.GraphDesc(pdf, obs).preorder()
    p = bm.registry().export_values()
    got, want = bm.eval_metric(p), ref.eval(p, 0)
    assert close(got, want), (got, want)
    for i, nd in enumerate(nodes):
        if isinstance(nd, pf.PolynomialPdf):
            assert nd.clamp_count() == ref.clamp_count(i) > 0, (nd.name(), nd.clamp_count(), ref.clamp_count(i))


def test_c5_dalitz_vs_oracle():
    """C5 shape: DalitzPlotPdf, 4 isobars, 2-D normalisation grid (128 here so
    the oracle's walk stays short).  No reference code: parity against the C
    restatement, itself checked against numpy in test_oracle.py."""
    W = WORKLOADS["C5TI"]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(20_011, seed=4))
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(128))
    o = oracle.Oracle(pdf, ds, 128)
    names = [p.name for p in bm.registry().parameters()]
    nodes = pf.GraphDesc(pdf, obs).preorder()
    bumped = dict(W.truth, rhom_re=0.5, rho0_im=0.3, f0_re=0.2)
    for pt in (W.start, W.truth, bumped):
        p = [pt[n] for n in names]
        got, want = bm.eval_metric(p), o.eval(p)
        assert close(got, want), (got, want)
        norms, _, valid = o.norms()
        assert valid[0] and close(nodes[0].cached_norm(), norms[0])


def test_device_partial_record_matches_host_partial():
    """pf_eval_launch + the device record (what bench.py all-gathers over NCCL
    on the model's stream) carry the same exact digits as pf_eval_partial"""
    import torch
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(21, 300_007))
    bm = pf.BoundModel(pdf, ds)
    p = [0.3, -0.8, 4.6, 1.3]
    fx, pen = bm.eval_partial(p)
    assert not pen

    class _Rec:
        def __init__(self, ptr):
            self.__cuda_array_interface__ = {"shape": (8,), "typestr": "<i8", "data": (ptr, False), "version": 3}

    rec = torch.as_tensor(_Rec(bm.partial_device()), device="cuda:0")
    stream = torch.cuda.ExternalStream(bm.stream(), device="cuda:0")
    p2 = [0.35, -0.7, 4.9, 1.1]
    want, _ = bm.eval_partial(p2)
    assert not bm.eval_launch(p)  # enqueued, not waited for
    with torch.cuda.stream(stream):
        got = rec.cpu().tolist()
    assert got[:6] == fx and got[6] == 0xFFFFFFFF and got[7] == 0
    assert bm.eval_launch([1.5, -0.7, 4.9, 1.1])  # invalid fraction: penalty, nothing enqueued
    assert bm.eval_partial(p2)[0] == want  # the host path stays in step after launches


def test_exchange_group_of_one_is_bitwise_the_plain_value():
    """the peer-memory exchange group (pf_group_join) with a single rank: the
    event pass stores its record into its own buffer, waits for it and sums
    the group's digits; the value must equal the ungrouped evaluation bit
    for bit, and keep doing so over repeated and batched calls"""
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * oracle.mt64_uniform(23, 200_003))
    plain = pf.BoundModel(pdf, ds)
    grouped = pf.BoundModel(pdf, ds)
    grouped.group_join(1, 0, [grouped.group_handle()])
    rng = np.random.default_rng(8)
    P = [[rng.uniform(0, 1), rng.uniform(-2, 0), rng.uniform(3, 7), rng.uniform(0.5, 2)] for _ in range(6)]
    for p in P:
        assert grouped.eval_metric(p) == plain.eval_metric(p)
    assert np.array_equal(grouped.eval_metric_batch(np.array(P)), plain.eval_metric_batch(np.array(P)))


def test_exchange_group_with_an_empty_shard():
    """a rank without events publishes through the publish kernel, which must
    take part in the exchange too (here: a group of one, empty data)"""
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], np.zeros(0))
    bm = pf.BoundModel(pdf, ds)
    bm.group_join(1, 0, [bm.group_handle()])
    assert bm.eval_metric([0.4, -0.6, 5.0, 1.0]) == 0.0
    assert bm.eval_metric([0.3, -0.5, 5.1, 1.1]) == 0.0


def test_c5_boundary_decisions_match_oracle():
    """Events within a few ulp of the Dalitz-plot boundary (both s13 limits,
    both s12 edges): the fast boundary test (pf_dalitz_inside_fast) decides
    every one like the oracle's exactly rounded sequence — a single flip would
    move the NLL by ~690 (floor) and the floor count."""
    W = WORKLOADS["C5TI"]
    obs, pdf = W.build(pf)
    M, (m1, m2, m3) = W.M, W.ms
    rng = np.random.default_rng(8)
    (a12, b12), _ = W.box()
    s12 = np.concatenate([rng.uniform(a12, b12, 3000),
                          a12 * (1 + np.arange(1, 40) * 2.0 ** -52), b12 * (1 - np.arange(1, 40) * 2.0 ** -52)])
    r12 = np.sqrt(s12)
    e1 = (s12 - m2 * m2 + m1 * m1) / (2 * r12)
    e3 = (M * M - s12 - m3 * m3) / (2 * r12)
    p1 = np.sqrt(np.maximum(e1 * e1 - m1 * m1, 0))
    p3 = np.sqrt(np.maximum(e3 * e3 - m3 * m3, 0))
    lo = (e1 + e3) ** 2 - (p1 + p3) ** 2
    hi = (e1 + e3) ** 2 - (p1 - p3) ** 2
    pts = []
    for k in range(-4, 5):
        pts.append(np.stack([s12, lo * (1 + k * 2.0 ** -52)]))
        pts.append(np.stack([s12, hi * (1 + k * 2.0 ** -52)]))
    cols = np.concatenate(pts, axis=1)
    _, (a13, b13) = W.box()
    cols = cols[:, (cols[1] >= a13) & (cols[1] <= b13)]
    ds = pf.UnbinnedDataSet.from_columns(obs, cols)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(64))
    o = oracle.Oracle(pdf, ds, 64)
    pt = dict(W.start, **W.truth)
    p = [pt[n.name] for n in bm.registry().parameters()]
    got, want = bm.eval_metric(p), o.eval(p)
    assert bm.log_floor_count() == o.floor_count() > 0
    assert close(got, want), (got, want)



def test_c4_batch_is_bitwise_sequential():
    """Convolution models stage the per-call state in shared memory (K x S
    must fit); a batch of parameter sets, including a resolution width that
    disables the term recurrence, equals the sequential calls bit for bit"""
    W = WORKLOADS["C4"]
    obs, pdf = W.build(pf)
    ds = W.data(pf, obs, 3000, seed=5)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
    names = [p.name for p in bm.registry().parameters()]
    pts = [W.start, W.truth, dict(m=2.9, w=0.35, rm=0.01, rs=0.06), dict(m=3.1, w=0.15, rm=-0.02, rs=0.0001)]
    P = np.array([[pt[n] for n in names] for pt in pts])
    batch = bm.eval_metric_batch(P, pf.MetricKind.ChiSquared)
    seq = np.array([bm.eval_metric(list(p), pf.MetricKind.ChiSquared) for p in P])
    assert np.array_equal(batch, seq)
    ref = oracle.Reference(pdf, ds, W.grid) if oracle.Reference.available() else oracle.Oracle(pdf, ds, W.grid)
    for p, got in zip(P, batch):
        assert close(got, ref.eval(list(p), 1)), (p, got)


def test_c4_wide_sums_and_nonfinite_index_match_reference():
    """chi-squared far from the data: chunk sums beyond 2^62 go through the
    wide accumulator (value still the reference's), and a non-finite term
    reports the reference's first offending bin (engine.hpp:210-216)"""
    W = WORKLOADS["C4"]
    obs, pdf = W.build(pf)
    ds = W.data(pf, obs, 3000, seed=5)
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(W.grid))
    ref = oracle.Reference(pdf, ds, W.grid) if oracle.Reference.available() else oracle.Oracle(pdf, ds, W.grid)
    wide = [2.5, 0.05, 0.2, 0.0001]
    got = bm.eval_metric(wide, pf.MetricKind.ChiSquared)
    want = ref.eval(wide, 1)
    assert want > 2.0 ** 64 and close(got, want), (got, want)
    truth = [W.truth[p.name] for p in bm.registry().parameters()]
    batch = bm.eval_metric_batch(np.array([wide, truth]), pf.MetricKind.ChiSquared)
    assert batch[0] == got and close(batch[1], ref.eval(truth, 1))
    bad = [3.5, 0.05, -0.2, 1e-5]
    with pytest.raises(Exception) as want_err:
        ref.eval(bad, 1)
    with pytest.raises(pf.Error) as got_err:
        bm.eval_metric(bad, pf.MetricKind.ChiSquared)
    assert str(got_err.value) == str(want_err.value)
    # the wide digits were reset: the next call is the plain one again
    assert bm.eval_metric(truth, pf.MetricKind.ChiSquared) == batch[1]


def test_c4_wide_sums_on_the_partial_path_raise_metric_overflow():
    """the cross-process partials carry only the six fixed-point digits: a
    shard whose chunk sums leave their range fails loudly (metric-overflow)
    instead of returning a wrong partial; in-range calls stay exact"""
    W = WORKLOADS["C4"]
    obs, pdf = W.build(pf)
    ds = W.data(pf, obs, 3000, seed=5)
    ref = oracle.Reference(pdf, ds, W.grid) if oracle.Reference.available() else oracle.Oracle(pdf, ds, W.grid)
    shards = [pf.BoundModel(pdf, ds, pf.GridSpec(W.grid), shard_index=r, shard_count=2) for r in range(2)]
    truth = [W.truth[p.name] for p in shards[0].registry().parameters()]
    parts = [bm.eval_partial(truth, pf.MetricKind.ChiSquared)[0] for bm in shards]
    assert close(pf.combine_partials(parts), ref.eval(truth, 1))
    with pytest.raises(pf.Error, match="metric-overflow"):
        for bm in shards:
            bm.eval_partial([2.5, 0.05, 0.2, 0.0001], pf.MetricKind.ChiSquared)
    parts2 = [bm.eval_partial(truth, pf.MetricKind.ChiSquared)[0] for bm in shards]
    assert [list(p) for p in parts2] == [list(p) for p in parts]


@pytest.mark.parametrize("n_dev", [2, 4, 8])
def test_multi_device_path_bitwise_on_oversubscribed_devices(n_dev):
    """the in-process multi-device path (engine.cpp: one shard per device,
    contiguous subtrees of the chunk range, host combine of the exact digits)
    run with its shards placed round-robin on the visible devices: bitwise
    the single-device value, for NLL, batched NLL and binned chi2 (no kernel
    waits on another, so sharing one GPU is safe)"""
    x, pdf = mixture()
    rng = np.random.default_rng(21)
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * rng.random(1_000_003))
    one = pf.BoundModel(pdf, ds)
    many = pf.BoundModel(pdf, ds, pf.GridSpec(), pf.Backend.gpus(n_dev, oversubscribe=True))
    p = one.registry().export_values()
    assert many.eval_metric(p) == one.eval_metric(p)
    assert many.log_floor_count() == one.log_floor_count()
    pts = np.array([p, [0.3, -0.5, 4.9, 1.1], [0.5, -0.7, 5.2, 0.9]])
    assert np.array_equal(many.eval_metric_batch(pts), one.eval_metric_batch(pts))
    W = WORKLOADS["C4"]
    obs, cpdf = W.build(pf)
    b = W.data(pf, obs, 20_000, seed=3)
    c1 = pf.BoundModel(cpdf, b, pf.GridSpec(W.grid))
    cn = pf.BoundModel(cpdf, b, pf.GridSpec(W.grid), pf.Backend.gpus(n_dev, oversubscribe=True))
    q = c1.registry().export_values()
    assert cn.eval_metric(q, pf.MetricKind.ChiSquared) == c1.eval_metric(q, pf.MetricKind.ChiSquared)


def test_more_devices_than_visible_is_refused():
    import torch
    x, pdf = mixture()
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * np.random.default_rng(1).random(1000))
    with pytest.raises(pf.Error) as ei:
        pf.BoundModel(pdf, ds, pf.GridSpec(), pf.Backend.gpus(torch.cuda.device_count() * 2))
    assert ei.value.args[0].startswith("bad-backend")


@pytest.mark.parametrize("mix", [(0.4101, 0.0039, 0.0065), (0.41, 0.15, -0.12)])
def test_c5_tddp_vs_oracle(mix):
    """C5 (BASELINE config 5): TddpPdf over (m12^2, m13^2, t), separable 3-D
    normalisation on the GPU (8 Dalitz-grid + 8 time-grid component sums)
    against the C restatement (its separable sum pinned to the brute-force
    3-D walk in test_oracle.py, its density to numpy).  Parity unpinned by
    nature (no reference code)."""
    W = WORKLOADS["C5"]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(20011, seed=4))
    grid = 64
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    o = oracle.Oracle(pdf, ds, grid)
    names = [v.name for v in bm.registry().parameters()]
    assert names == o.param_names()
    p = [W.truth[n] for n in names]
    p[names.index("tau")], p[names.index("x")], p[names.index("y")] = mix
    got, want = bm.eval_metric(p), o.eval(p)
    assert close(got, want), (got, want, abs(got - want) / abs(want))
    assert close(pdf.cached_norm(), o.norms()[0][0])
    q = list(p)
    q[names.index("rhom_re")] *= 1.1
    assert close(bm.eval_metric(q), o.eval(q))
    # batched == sequential
    assert np.array_equal(bm.eval_metric_batch(np.array([p, q])), [bm.eval_metric(p), bm.eval_metric(q)])
    # tau <= 0: the normalisation fails -> the reference's penalty (engine.hpp:174-178)
    r = list(p)
    r[names.index("tau")] = -0.1
    assert bm.eval_metric(r) == o.eval(r) == pf.kPenaltyValue


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_small_grid_workloads_take_the_single_kernel_path(name):
    """C1-C3 (one parameter set, small normalisation grids) run as ONE fused
    kernel per call; a layout change that no longer fits it would silently
    fall back to the slower two-kernel graph"""
    W = WORKLOADS[name]
    obs, pdf = W.build(pf)
    bm = pf.BoundModel(pdf, W.data(pf, obs, 50_000, seed=2), pf.GridSpec(W.grid))
    bm.eval_metric(W.params(bm))
    assert pf.lib.pf_model_fused(bm._h) == 1


@pytest.mark.parametrize("name", ["C5", "C5TI"])
def test_dalitz_grid_column_tables_match_the_per_point_path(name, monkeypatch):
    """The Dalitz / TDDP normalisation grids take channel A (s13) from a
    per-block column table (pf_tddp_cols / pf_dalitz_cols); with the table
    off (PFB200_NOTDDPTAB) every point evaluates it.  Both agree to rounding
    and with the oracle, for one parameter set and a batch."""
    W = WORKLOADS[name]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(20011, seed=6))
    grid = 128
    on = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    monkeypatch.setenv("PFB200_NOTDDPTAB", "1")
    off = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    monkeypatch.delenv("PFB200_NOTDDPTAB")
    o = oracle.Oracle(pdf, ds, grid)
    names = [v.name for v in on.registry().parameters()]
    p = [W.truth[n] for n in names]
    q = list(p)
    q[names.index("rhop_re" if "rhop_re" in names else names[2])] *= 0.9
    for x in (p, q):
        a, b, want = on.eval_metric(x), off.eval_metric(x), o.eval(x)
        assert abs(a - b) <= 1e-14 * abs(b), (a, b)
        assert close(a, want), (a, want)
    assert np.array_equal(on.eval_metric_batch(np.array([p, q])), [on.eval_metric(p), on.eval_metric(q)])


def test_tddp_models_of_different_grids_share_a_module():
    """Two TddpPdf models of one structure share the compiled module and its
    norm-kernel shared-memory limit; the larger grid's column table must not
    break the smaller one's launches, whichever is created first"""
    W = WORKLOADS["C5"]
    obs, pdf = W.build(pf)
    ds = pf.UnbinnedDataSet.from_columns(obs, W.columns(5003, seed=8))
    big = pf.BoundModel(pdf, ds, pf.GridSpec(256))
    small = pf.BoundModel(pdf, ds, pf.GridSpec(64))
    p = big.registry().export_values()
    a, b = big.eval_metric(p), small.eval_metric(p)
    assert np.isfinite(a) and np.isfinite(b)
    assert big.eval_metric(p) == a and small.eval_metric(p) == b
    o = oracle.Oracle(pdf, ds, 256)
    assert close(a, o.eval(p))
