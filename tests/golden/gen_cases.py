"""Toy-generation catalogue: the reference's own generate_events calls
(file:line per case) as (pdf, observables, n_events, seed, grid).  Used by
make_generate_golden.py (the compiled reference, oracle/_ref) and by
tests/test_gpu_generate.py (the GPU generator)."""


def gen_exp_seed42(pf):
    """test_generate.cpp:37-47: Exp(a=-0.5) on [0, 10], 2000 events, seed 42"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.5, 0.1, -5, 5)
    return pf.exp_pdf("e", x, a), [x], 2000, 42, 1024


def gen_exp_seed43(pf):
    """test_generate.cpp:46: the same with seed 43 (must differ)"""
    pdf, obs, n, _, grid = gen_exp_seed42(pf)
    return pdf, obs, n, 43, grid


def gen_uniform(pf):
    """test_generate.cpp:50-67: constant polynomial on [2, 8], 20000 events, seed 11"""
    x = pf.new_observable("x", 2, 8)
    c0 = pf.new_parameter("c0", 1, 0.1, 0.5, 2)
    return pf.polynomial_pdf("u", x, [c0]), [x], 20000, 11, 1024


def gen_exp_cdf(pf):
    """test_generate.cpp:69-87: Exp(a=-0.7) on [0, 10], 40000 events, seed 2024"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.7, 0.1, -5, 5)
    return pf.exp_pdf("e", x, a), [x], 40000, 2024, 1024


def gen_gauss(pf):
    """test_generate.cpp:89-104: Gauss(1.2, 0.8) on [-6, 6], 30000 events, seed 5"""
    x = pf.new_observable("x", -6, 6)
    m = pf.new_parameter("m", 1.2, 0.1, -4, 4)
    s = pf.new_parameter("s", 0.8, 0.1, 0.1, 3)
    return pf.gaussian_pdf("g", x, m, s), [x], 30000, 5, 1024


def gen_prod2d(pf):
    """test_generate.cpp:106-126: Exp(x)·Exp(y) on [0, 5]^2, 30000 events, seed 99"""
    x = pf.new_observable("x", 0, 5)
    y = pf.new_observable("y", 0, 5)
    ax = pf.new_parameter("ax", -2.4, 0.1, -5, 5)
    ay = pf.new_parameter("ay", -1.1, 0.1, -5, 5)
    pdf = pf.prod_pdf("p", [pf.exp_pdf("ex", x, ax), pf.exp_pdf("ey", y, ay)])
    return pdf, [x, y], 30000, 99, 1024


def gen_closure(pf):
    """test_generate.cpp:128-139: Exp(a=-0.7) on [0, 10], 20000 events, seed 314"""
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -0.7, 0.2, -5, -0.05)
    return pf.exp_pdf("gen", x, a), [x], 20000, 314, 1024


def gen_criterion1(pf):
    """acceptance.cpp:85-88: Exp(alpha=-2) on [0, 21.49], 1e5 events, seed 20260823"""
    x = pf.new_observable("xvar", 0, 21.49)
    a = pf.new_parameter("alpha", -2, 0.5, -10, 10)
    return pf.exp_pdf("gen", x, a), [x], 100000, 20260823, 1024


def gen_criterion2(pf):
    """acceptance.cpp:116-123: Exp(x)·Exp(y) on [0, 5]^2, 50000 events, seed 77, grid 512"""
    x = pf.new_observable("x", 0, 5)
    y = pf.new_observable("y", 0, 5)
    gx = pf.new_parameter("ax", -2.4, 0.3, -8, 8)
    gy = pf.new_parameter("ay", -1.1, 0.3, -8, 8)
    pdf = pf.prod_pdf("gen", [pf.exp_pdf("gx", x, gx), pf.exp_pdf("gy", y, gy)])
    return pdf, [x, y], 50000, 77, 512


def gen_bw(pf):
    """acceptance.cpp:386-395: Breit-Wigner(3.0, 0.2) on [2, 4], 130000 events, seed 99"""
    x = pf.new_observable("xg", 2, 4)
    m = pf.new_parameter("mg", 3.0, 0.01, 2, 4)
    w = pf.new_parameter("wg", 0.2, 0.01, 0.01, 1)
    return pf.breit_wigner_pdf("bw", x, m, w), [x], 130000, 99, 1024


def gen_mixture(pf):
    """BASELINE C2's proposed input: f Gauss(5, 0.8) + Exp(-0.6)
    on [0, 10] at truth, seed 11 (200000 events here)"""
    x = pf.new_observable("x", 0, 10)
    m = pf.new_parameter("m", 5.0, 0.1, 0, 10)
    s = pf.new_parameter("s", 0.8, 0.1, 0.1, 5)
    a = pf.new_parameter("a", -0.6, 0.1, -5, 5)
    f = pf.new_parameter("f", 0.3, 0.01, 0, 1)
    pdf = pf.add_pdf("sigbkg", [pf.gaussian_pdf("sig", x, m, s), pf.exp_pdf("bkg", x, a)], [f])
    return pdf, [x], 200000, 11, 1024


def gen_composite_mapped(pf):
    """Composite Gauss(u) of Exp(x) and a MappedPdf: the synthetic column and
    the boundary search inside the accept test (pdf.hpp:406-452)"""
    x = pf.new_observable("x", 0, 10)
    u = pf.new_observable("u", 0, 1)
    a = pf.new_parameter("a", -0.5, 0.1, -10, 10)
    m = pf.new_parameter("m", 0.25, 0.1, -5, 5)
    s = pf.new_parameter("s", 0.3, 0.1, 0.01, 5)
    comp = pf.composite_pdf("comp", pf.gaussian_pdf("g", u, m, s), pf.exp_pdf("inner", x, a))
    b = pf.new_parameter("b", -0.2, 0.1, -5, 5)
    mapped = pf.mapped_pdf("map", [0, 4, 10], [comp, pf.exp_pdf("tail", x, b)])
    return mapped, [x], 20000, 7, 1024


def gen_extra_observable(pf):
    """an observable outside the PDF's box keeps its current value in every
    event (generate.hpp:79 sets only box observables; add_event snapshots all)"""
    x = pf.new_observable("x", 0, 10)
    z = pf.new_observable("z", -1, 1)
    z.value = 0.375
    a = pf.new_parameter("a", -0.4, 0.1, -5, 5)
    return pf.exp_pdf("e", x, a), [x, z], 5000, 3, 1024


def restated_generate(pf, pdf, obs, n, seed, grid):
    """generate.hpp:33-86 restated over the C oracle's densities and the
    ToyRng stream (test infrastructure)"""
    import numpy as np

    import oracle
    dummy = pf.UnbinnedDataSet.from_columns(obs, np.array([[o.lower] for o in obs]))
    orc = oracle.Oracle(pdf, dummy, grid)
    p = [orc.desc.vars[orc.L.po_param_variable(orc.h, i)].value for i in range(orc.L.po_n_params(orc.h))]
    d = len(obs)  # every case here has all observables in the box, in obs order
    h = [(o.upper - o.lower) / grid for o in obs]
    k = np.indices((grid,) * d).reshape(d, -1).astype(np.float64)
    mids = np.stack([obs[i].lower + (k[i] + 0.5) * h[i] for i in range(d)])
    dens = orc.density(p, mids)
    dmax = float(np.max(np.where(dens > 0, dens, 0.0)))
    env = dmax * 1.1
    taken, cand0, out = 0, 0, []
    while taken < n:
        m = 200_000
        u = oracle.mt64_uniform(seed, (cand0 + m) * (d + 1))[cand0 * (d + 1):].reshape(m, d + 1)
        pts = np.stack([obs[i].lower + (obs[i].upper - obs[i].lower) * u[:, i] for i in range(d)])
        dn = orc.density(p, pts)
        assert not np.any(dn > env), "restatement: envelope failure"
        acc = u[:, d] * env < dn
        out.append(pts[:, acc])
        taken += int(acc.sum())
        cand0 += m
    return np.concatenate(out, axis=1)[:, :n]


CASES = {k[4:]: v for k, v in dict(globals()).items() if k.startswith("gen_")}
