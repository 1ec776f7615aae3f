"""Golden-case catalogue: models and seeded data sets mirroring the
reference's own tests (file:line cited per case).  Used by make_golden.py
(which evaluates them with the compiled reference, oracle/_ref) and by the
parity tests (which evaluate them with the C oracle and the GPU engine).

Data are regenerated deterministically from std::mt19937_64 draws
(oracle.mt64_uniform, the reference's uniform01 / ToyRng recipe), so only
the expected values are stored in golden.json.
"""
import math

import numpy as np


def _u(seed, n):
    import oracle
    return oracle.mt64_uniform(seed, n)


def exp_toy(pf, x, alpha, n, seed):
    """test_fit.cpp:19-32 make_exp_toy (inverse transform on [0, upper])"""
    u = _u(seed, n)
    return pf.UnbinnedDataSet.from_columns([x], np.log(1.0 + u * (np.exp(alpha * x.upper) - 1.0)) / alpha)


def box_muller(seed, n, cut=5.0):
    """test_fit.cpp:176-187 (truth mean 0, sigma 1, |z| < cut)"""
    u = _u(seed, 4 * n + 16)
    out, i = [], 0
    while len(out) < n:
        u1, u2 = u[i], u[i + 1]
        i += 2
        if u1 <= 0:
            continue
        z = math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2)
        if abs(z) >= cut:
            continue
        out.append(z)
    return np.array(out)


def case_listing1(pf):
    """Listing 1 / test_fit.cpp:156-169: ExpPdf on [0, 21.49], alpha = -2."""
    x = pf.new_observable("xvar", 0, 21.49)
    alpha = pf.new_parameter("alpha", -1.0, 0.5, -10, 10)
    ds = exp_toy(pf, x, -2.0, 20000, 1234)
    return pf.exp_pdf("exppdf", x, alpha), ds, 1024, [[-2.0], [-1.5], [-2.5], [-1.0]]


def case_mixture_acceptance(pf):
    """acceptance.cpp:305-348: 1e6 events, mt19937_64(31), NLL 3218448.5501374062."""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.6, 0.1, -5, 5)
    m = pf.new_parameter("m", 5, 0.1, 0, 10)
    s = pf.new_parameter("s", 1, 0.1, 0.1, 5)
    f = pf.new_parameter("f", 0.4, 0.01, 0, 1)
    pdf = pf.add_pdf("mix", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s)], [f])
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * _u(31, 1_000_000))
    return pdf, ds, 1024, [[0.4, -0.6, 5, 1], [0.2, -1.1, 4.5, 0.7], [0.9, -0.05, 6.5, 2.5]]


def case_product2d(pf):
    """acceptance.cpp:117-152 / test_pdf.cpp:169-185: Prod(Exp(x), Exp(y)), grid 512."""
    x = pf.new_observable("x", 0, 5)
    y = pf.new_observable("y", 0, 5)
    ax = pf.new_parameter("ax", -2.4, 0.3, -8, 8)
    ay = pf.new_parameter("ay", -1.1, 0.3, -8, 8)
    pdf = pf.prod_pdf("prod", [pf.exp_pdf("ex", x, ax), pf.exp_pdf("ey", y, ay)])
    u = _u(77, 2 * 30000)
    ds = pf.UnbinnedDataSet.from_columns([x, y], np.stack([5 * u[0::2], 5 * u[1::2]]))
    return pdf, ds, 512, [[-2.4, -1.1], [-1.5, -0.5], [0.3, 0.2]]


def case_gauss_fit(pf):
    """test_fit.cpp:171-194: Gaussian mean/sigma on Box-Muller data."""
    x = pf.new_observable("x", -5, 5)
    mean = pf.new_parameter("mean", 0.3, 0.5, -4, 4)
    sigma = pf.new_parameter("sigma", 1.1, 0.5, 0.2, 4)
    ds = pf.UnbinnedDataSet.from_columns([x], box_muller(99, 4000))
    return pf.gaussian_pdf("g", x, mean, sigma), ds, 1024, [[0.3, 1.1], [0.0, 1.0], [-0.2, 0.9]]


def case_three_mixture(pf):
    """test_engine.cpp:168-186 shape with valid fractions: 3 children, 2 fractions."""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.3, 0.1, -10, 10)
    m = pf.new_parameter("m", 5, 0.1, 0, 10)
    s = pf.new_parameter("s", 1, 0.1, 0.1, 5)
    s2 = pf.new_parameter("s2", 2.5, 0.1, 0.1, 5)
    f1 = pf.new_parameter("f1", 0.3, 0.01, 0, 1)
    f2 = pf.new_parameter("f2", 0.2, 0.01, 0, 1)
    pdf = pf.add_pdf("mix3", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s),
                              pf.gaussian_pdf("g2", x, m, s2)], [f1, f2])
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * _u(5, 50000))
    return pdf, ds, 1024, [[0.3, 0.2, -0.3, 5, 1, 2.5], [0.6, 0.1, -0.8, 4.0, 0.5, 1.5]]


def case_polynomial(pf):
    """test_engine.cpp:150-166 / test_pdf.cpp:146-167: ramp with clamping."""
    x = pf.new_observable("x", 0, 10)
    c0 = pf.new_parameter("c0", 1.0, 0.1, -5, 5)
    c1 = pf.new_parameter("c1", -0.05, 0.1, -5, 5)
    c2 = pf.new_parameter("c2", 0.002, 0.001, -5, 5)
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * _u(11, 20000))
    return pf.polynomial_pdf("poly", x, [c0, c1, c2]), ds, 1024, [[1.0, -0.05, 0.002],
                                                                  [1.0, -0.3, 0.01]]


def case_breit_wigner(pf):
    """test_pdf.cpp:106-144: BreitWignerPdf on [0.5, 1.5]."""
    x = pf.new_observable("x", 0.5, 1.5)
    mass = pf.new_parameter("m", 1.0, 0.01, 0.6, 1.4)
    width = pf.new_parameter("w", 0.05, 0.001, 0.001, 0.5)
    ds = pf.UnbinnedDataSet.from_columns([x], 0.5 + _u(21, 20000))
    return pf.breit_wigner_pdf("bw", x, mass, width), ds, 1024, [[1.0, 0.05], [0.9, 0.2]]


def case_mapped(pf):
    """test_pdf.cpp:339-367: piecewise {Exp on [0,5), Gauss on [5,10]}."""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.8, 0.1, -10, 10)
    m = pf.new_parameter("m", 7, 0.1, 0, 10)
    s = pf.new_parameter("s", 0.9, 0.1, 0.01, 5)
    pdf = pf.mapped_pdf("pw", [0, 5, 10], [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s)])
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * _u(23, 20000))
    return pdf, ds, 1024, [[-0.8, 7, 0.9], [-0.2, 6.0, 1.5]]


def case_composite(pf):
    """test_pdf.cpp:276-306: composite Gauss(u) of Exp(x)."""
    x = pf.new_observable("x", 0, 10)
    u = pf.new_observable("u", 0, 1)
    a = pf.new_parameter("a", -0.5, 0.1, -10, 10)
    m = pf.new_parameter("m", 0.25, 0.1, -5, 5)
    s = pf.new_parameter("s", 0.3, 0.1, 0.01, 5)
    pdf = pf.composite_pdf("comp", pf.gaussian_pdf("g", u, m, s), pf.exp_pdf("inner", x, a))
    ds = pf.UnbinnedDataSet.from_columns([x], 10.0 * _u(29, 20000))
    return pdf, ds, 1024, [[0.25, 0.3, -0.5], [0.1, 0.5, -0.2]]


def case_convolution(pf):
    """test_pdf.cpp:385-402: Gauss (x) Gauss, Q = 256, grid 256, unbinned."""
    x = pf.new_observable("x", -10, 10)
    m1 = pf.new_parameter("m1", 0, 0.1, -5, 5)
    s1 = pf.new_parameter("s1", 0.8, 0.01, 0.01, 5)
    m2 = pf.new_parameter("m2", 0, 0.1, -5, 5)
    s2 = pf.new_parameter("s2", 0.6, 0.01, 0.01, 5)
    pdf = pf.convolution_pdf("conv", pf.gaussian_pdf("g1", x, m1, s1), pf.gaussian_pdf("g2", x, m2, s2), 256)
    ds = pf.UnbinnedDataSet.from_columns([x], box_muller(37, 3000, cut=5.0) * 1.0)
    return pdf, ds, 256, [[0, 0.8, 0, 0.6], [0.2, 1.1, 0.0, 0.4]]


def case_bw_conv_binned(pf):
    """acceptance.cpp:386-433 (criterion 7): BW (x) Gauss, binned chi2, 200 bins,
    Q = 64, grid 256, resolution parameters fixed."""
    x = pf.new_observable("x", 2, 4)
    m = pf.new_parameter("m", 3.05, 0.05, 2.5, 3.5)
    w = pf.new_parameter("w", 0.3, 0.05, 0.05, 0.6)
    rm = pf.new_parameter("rm", 0.0, 0.01, -0.2, 0.2)
    rs = pf.new_parameter("rs", 0.05, 0.01, 0.02, 0.15)
    rm.fixed = True
    rs.fixed = True
    pdf = pf.convolution_pdf("sig", pf.breit_wigner_pdf("bw", x, m, w), pf.gaussian_pdf("res", x, rm, rs), 64)
    # smeared Breit-Wigner toy contents (deterministic, no accept-reject):
    # inverse-CDF of a Cauchy in x^2 around m=3.0, w=0.2, then Gaussian noise
    u = _u(99, 200000)
    z = box_muller(100, 100000)
    xs = []
    k = 0
    for i in range(100000):
        t = math.tan(math.pi * (u[i] - 0.5))
        v = 3.0 + 0.1 * t + 0.05 * z[i]
        if 2 <= v <= 4:
            xs.append(v)
    b = pf.BinnedDataSet([x], [200])
    counts, _ = np.histogram(np.array(xs), bins=200, range=(2.0, 4.0))
    b.set_contents(counts.astype(np.float64))
    del k
    return pdf, b, 256, [[3.05, 0.3, 0.0, 0.05], [3.0, 0.2, 0.0, 0.05]]


CASES = {
    "listing1": case_listing1,
    "mixture_acceptance": case_mixture_acceptance,
    "product2d": case_product2d,
    "gauss_fit": case_gauss_fit,
    "three_mixture": case_three_mixture,
    "polynomial": case_polynomial,
    "breit_wigner": case_breit_wigner,
    "mapped": case_mapped,
    "composite": case_composite,
    "convolution": case_convolution,
    "bw_conv_binned": case_bw_conv_binned,
}

# cases whose reference fit() result is stored too (small enough for CPU)
FIT_CASES = ["listing1", "gauss_fit", "product2d", "bw_conv_binned"]
