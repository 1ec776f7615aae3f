"""The BASELINE.json configurations as concrete, seeded workloads (SURVEY.md
§8(d)): model builders over the parfit mirror, synthetic data of each
config's shape (numpy, deterministic), start points and the algorithmic
bytes per unit that the roofline uses.

  C1  ExpPdf on [0, 21.49], the paper's listing (CPU-sized)
  C2  AddPdf(GaussianPdf, ExpPdf), 1e7 events per GPU (bench default)
  C3  ProdPdf(GaussianPdf(x), ArgusPdf(y)), 1e8 events (sharded)
  C4  ConvolutionPdf(BreitWigner, Gaussian), binned chi-squared, 1e6 bins

Data are synthetic (no network): numpy PCG64 streams with fixed seeds.
"""
from __future__ import annotations

import numpy as np


class Workload:
    name = ""
    description = ""
    metric = 0            # parfit MetricKind: 0 NLL, 1 chi-squared
    unit = "events"
    default_n = 0         # events (bins) per GPU for weak scaling, total for strong
    scaling = "weak"
    grid = 1024
    fit_n = 100_000       # events (bins) of the full-fit wall-time comparison
    has_reference = True  # False: a PDF the reference lacks (CPU legs use the C restatement)
    start: dict = {}
    truth: dict = {}

    def build(self, pf):
        """-> (observables, pdf) with parameters at the start point"""
        raise NotImplementedError

    def data(self, pf, observables, n, seed=11):
        raise NotImplementedError

    def bytes_per_unit(self):
        """algorithmic HBM bytes per event (bin): the EventTable columns read"""
        raise NotImplementedError

    def params(self, bm):
        return np.array([self.start[p.name] for p in bm.registry().parameters()])


def _trunc_normal(rng, mu, sigma, lo, hi, n):
    x = rng.normal(mu, sigma, n)
    bad = (x < lo) | (x > hi)
    while bad.any():
        x[bad] = rng.normal(mu, sigma, int(bad.sum()))
        bad = (x < lo) | (x > hi)
    return x


def _trunc_exp(u, a, hi):
    """inverse CDF of exp(a x) on [0, hi]"""
    return np.log1p(u * np.expm1(a * hi)) / a


class C1(Workload):
    name = "C1"
    description = "ExpPdf on [0, 21.49] (paper listing), alpha fit from -1"
    default_n = 100_000
    start = dict(alpha=-1.0)
    truth = dict(alpha=-2.0)

    def build(self, pf):
        x = pf.new_observable("xvar", 0.0, 21.49)
        alpha = pf.new_parameter("alpha", self.start["alpha"], 0.5, -10, 10)
        return [x], pf.exp_pdf("exppdf", x, alpha)

    @classmethod
    def columns(cls, n, seed=11):
        rng = np.random.default_rng(seed)
        return _trunc_exp(rng.random(n), cls.truth["alpha"], 21.49)

    def data(self, pf, obs, n, seed=11):
        return pf.UnbinnedDataSet.from_columns(obs, self.columns(n, seed))

    def bytes_per_unit(self):
        return 8.0


class C2(Workload):
    name = "C2"
    description = "AddPdf(GaussianPdf, ExpPdf) unbinned NLL on x in [0, 10]"
    default_n = 10_000_000
    start = dict(m=4.8, s=1.0, a=-0.5, f=0.4)
    truth = dict(m=5.0, s=0.8, a=-0.6, f=0.3)

    def build(self, pf):
        x = pf.new_observable("x", 0.0, 10.0)
        m = pf.new_parameter("m", self.start["m"], 0.1, 0.0, 10.0)
        s = pf.new_parameter("s", self.start["s"], 0.1, 0.1, 5.0)
        a = pf.new_parameter("a", self.start["a"], 0.1, -5.0, 5.0)
        f = pf.new_parameter("f", self.start["f"], 0.01, 0.0, 1.0)
        pdf = pf.add_pdf("sigbkg", [pf.gaussian_pdf("sig", x, m, s), pf.exp_pdf("bkg", x, a)], [f])
        return [x], pdf

    @classmethod
    def columns(cls, n, seed=11):
        """f Gauss(5, 0.8) + (1 - f) Exp(-0.6), truncated to [0, 10]"""
        t = cls.truth
        rng = np.random.default_rng(seed)
        u = rng.random(n)
        sig = rng.random(n) < t["f"]
        xe = _trunc_exp(u, t["a"], 10.0)
        xg = _trunc_normal(rng, t["m"], t["s"], 0.0, 10.0, n)
        return np.where(sig, xg, xe)

    def data(self, pf, obs, n, seed=11):
        return pf.UnbinnedDataSet.from_columns(obs, self.columns(n, seed))

    def bytes_per_unit(self):
        return 8.0


def argus_density(y, m0, c, p):
    """ARGUS shape y (1 - (y/m0)^2)^p exp(c (1 - (y/m0)^2)), 0 at and above m0"""
    t = 1.0 - (y / m0) ** 2
    out = np.zeros_like(y)
    ok = t > 0
    out[ok] = y[ok] * t[ok] ** p * np.exp(c * t[ok])
    return out


class C3(Workload):
    name = "C3"
    description = "ProdPdf(GaussianPdf(x), ArgusPdf(y)), x in [0, 10], y in [5.20, 5.29]"
    default_n = 100_000_000
    scaling = "strong"
    has_reference = False  # ArgusPdf
    start = dict(m=4.9, s=1.05, m0=5.29, c=-19.0, p=0.55)
    truth = dict(m=5.0, s=1.0, m0=5.29, c=-20.0, p=0.5)
    ylo, yhi = 5.20, 5.29

    def build(self, pf):
        x = pf.new_observable("x", 0.0, 10.0)
        y = pf.new_observable("y", self.ylo, self.yhi)
        m = pf.new_parameter("m", self.start["m"], 0.1, 0.0, 10.0)
        s = pf.new_parameter("s", self.start["s"], 0.05, 0.1, 5.0)
        m0 = pf.new_parameter("m0", self.start["m0"], 0.001, 5.28, 5.30)
        m0.fixed = True
        c = pf.new_parameter("c", self.start["c"], 0.5, -60.0, 0.0)
        p = pf.new_parameter("p", self.start["p"], 0.05, 0.05, 2.0)
        pdf = pf.prod_pdf("sigxy", [pf.gaussian_pdf("gx", x, m, s), pf.argus_pdf("argy", y, m0, c, p)])
        return [x, y], pdf

    @classmethod
    def columns(cls, n, seed=11):
        t = cls.truth
        rng = np.random.default_rng(seed)
        x = _trunc_normal(rng, t["m"], t["s"], 0.0, 10.0, n)
        grid = np.linspace(cls.ylo, cls.yhi, 20001)
        fmax = argus_density(grid, t["m0"], t["c"], t["p"]).max() * 1.01
        y = np.empty(n)
        filled = 0
        while filled < n:  # accept-reject, vectorised in blocks
            k = min(2 * (n - filled) + 1024, 1 << 24)
            cand = cls.ylo + (cls.yhi - cls.ylo) * rng.random(k)
            keep = cand[rng.random(k) * fmax < argus_density(cand, t["m0"], t["c"], t["p"])]
            take = min(len(keep), n - filled)
            y[filled:filled + take] = keep[:take]
            filled += take
        return np.stack([x, y])

    def data(self, pf, obs, n, seed=11):
        return pf.UnbinnedDataSet.from_columns(obs, self.columns(n, seed))

    def bytes_per_unit(self):
        return 16.0


class C4(Workload):
    name = "C4"
    description = ("ConvolutionPdf(BreitWignerPdf, GaussianPdf) binned chi-squared on x in [2, 4], "
                   "Q = 1024, resolution fixed")
    metric = 1
    unit = "bins"
    default_n = 1_000_000
    fit_n = 10_000
    q = 1024
    start = dict(m=3.05, w=0.25, rm=0.0, rs=0.05)
    truth = dict(m=3.0, w=0.2, rm=0.0, rs=0.05)
    total = 1e8

    def build(self, pf):
        x = pf.new_observable("x", 2.0, 4.0)
        m = pf.new_parameter("m", self.start["m"], 0.05, 2.5, 3.5)
        w = pf.new_parameter("w", self.start["w"], 0.05, 0.05, 0.6)
        rm = pf.new_parameter("rm", self.start["rm"], 0.01, -0.2, 0.2)
        rs = pf.new_parameter("rs", self.start["rs"], 0.01, 0.02, 0.15)
        rm.fixed = True
        rs.fixed = True
        pdf = pf.convolution_pdf("sig", pf.breit_wigner_pdf("bw", x, m, w), pf.gaussian_pdf("res", x, rm, rs),
                                 self.q)
        return [x], pdf

    @classmethod
    def contents(cls, n_bins, seed=11):
        """BW(3.0, 0.2) smeared by N(0, 0.05) (FFT convolution on the bin grid),
        scaled to ~1e8 entries, Poisson-fluctuated"""
        t = cls.truth
        edges = np.linspace(2.0, 4.0, n_bins + 1)
        xc = 0.5 * (edges[:-1] + edges[1:])
        h = edges[1] - edges[0]
        bw = 1.0 / ((xc * xc - t["m"] ** 2) ** 2 + t["m"] ** 2 * t["w"] ** 2)
        from scipy.signal import fftconvolve
        half = min(n_bins // 2, int(np.ceil(8 * t["rs"] / h)))
        g = np.exp(-0.5 * (np.arange(-half, half + 1) * h / t["rs"]) ** 2)
        sm = np.clip(fftconvolve(bw, g, mode="same"), 0.0, None)
        mu = cls.total * sm / sm.sum()
        return np.random.default_rng(seed).poisson(mu).astype(np.float64)

    def data(self, pf, obs, n, seed=11):
        b = pf.BinnedDataSet(obs, [n])
        b.set_contents(self.contents(n, seed))
        return b

    def bytes_per_unit(self):
        return 24.0  # EventTable row: bin centre, content, volume (dataset.hpp:161-182)


def dalitz_inside(s12, s13, M, ms):
    """the kinematic boundary of M -> 1 2 3 in the 12 rest frame"""
    m1, m2, m3 = ms
    r12 = np.sqrt(np.clip(s12, 1e-300, None))
    e1 = (s12 - m2 * m2 + m1 * m1) / (2 * r12)
    e3 = (M * M - s12 - m3 * m3) / (2 * r12)
    p1 = np.sqrt(np.clip(e1 * e1 - m1 * m1, 0, None))
    p3 = np.sqrt(np.clip(e3 * e3 - m3 * m3, 0, None))
    lo = (e1 + e3) ** 2 - (p1 + p3) ** 2
    hi = (e1 + e3) ** 2 - (p1 - p3) ** 2
    return (s12 >= (m1 + m2) ** 2) & (s12 <= (M - m3) ** 2) & (s13 >= lo) & (s13 <= hi)


def dalitz_amplitude(s12, s13, s23, M, ms, R, res):
    """numpy complex isobar amplitude at (s12, s13, s23), boundary aside (an
    independent copy of the formulas in pf_device.cuh / pf_oracle.c)"""
    m1, m2, m3 = ms
    mm = {1: m1, 2: m2, 3: m3}

    def q2(s, a, b):
        return np.clip((s - (a + b) ** 2) * (s - (a - b) ** 2) / (4 * s), 0, None)

    A = np.zeros_like(np.asarray(s12, dtype=np.float64), dtype=np.complex128)
    for mass, width, cre, cim, ch, spin in res:
        i, j = ch // 10, ch % 10
        k = 6 - i - j
        sv = {12: s12, 13: s13, 23: s23}
        sij = sv[ch]
        sik = sv[int(f"{min(i, k)}{max(i, k)}")]
        sjk = sv[int(f"{min(j, k)}{max(j, k)}")]
        qq = q2(sij, mm[i], mm[j])
        q0 = q2(mass * mass, mm[i], mm[j])
        x = np.sqrt(qq) / np.sqrt(q0)
        if spin == 1:
            bf2 = (1 + R * R * q0) / (1 + R * R * qq)
            ratio = x ** 3
            Z = sjk - sik + (M * M - mm[k] ** 2) * (mm[i] ** 2 - mm[j] ** 2) / sij
        else:
            bf2, ratio, Z = 1.0, x, 1.0
        g = width * ratio * mass / np.sqrt(sij) * bf2
        A += complex(cre, cim) * Z * np.sqrt(bf2) / (mass * mass - sij - 1j * mass * g)
    return A


def tddp_density(s12, s13, t, M, ms, R, res, tau, x, y):
    """numpy TddpPdf density (pfb200.h): |A g+ + Abar g-|^2 with
    Abar(s12, s13) = A(s12, s23), computed from its complex form"""
    m1, m2, m3 = ms
    s12 = np.asarray(s12, dtype=np.float64)
    s13 = np.asarray(s13, dtype=np.float64)
    s23 = M * M + m1 * m1 + m2 * m2 + m3 * m3 - s12 - s13
    A = dalitz_amplitude(s12, s13, s23, M, ms, R, res)
    Ab = dalitz_amplitude(s12, s23, s13, M, ms, R, res)
    T = np.asarray(t, dtype=np.float64) / tau
    # g+- = (e^{-i l1 t} +- e^{-i l2 t}) / 2 with l12 = (1 +- x)/tau... in units of 1/tau:
    # |g+|^2 = e^-T (cosh yT + cos xT)/2, |g-|^2 = e^-T (cosh yT - cos xT)/2,
    # g+* g- = e^-T (-sinh yT + i sin xT)/2 -- the convention of pfb200.h
    gp2 = np.exp(-T) * (np.cosh(y * T) + np.cos(x * T)) / 2
    gm2 = np.exp(-T) * (np.cosh(y * T) - np.cos(x * T)) / 2
    gpgm = np.exp(-T) * (-np.sinh(y * T) + 1j * np.sin(x * T)) / 2
    v = np.abs(A) ** 2 * gp2 + np.abs(Ab) ** 2 * gm2 + 2 * np.real(np.conj(A) * Ab * gpgm)
    return np.where(dalitz_inside(s12, s13, M, ms), v, 0.0)


def dalitz_amplitude2(s12, s13, M, ms, R, res):
    """numpy |A|^2 of the isobar model (the generator's copy of the kernels in
    pf_device.cuh / pf_oracle.c; used only to draw toy events)"""
    m1, m2, m3 = ms
    mm = {1: m1, 2: m2, 3: m3}
    s12 = np.asarray(s12, dtype=np.float64)
    s13 = np.asarray(s13, dtype=np.float64)
    s23 = M * M + m1 * m1 + m2 * m2 + m3 * m3 - s12 - s13
    # kinematic boundary (12 rest frame)
    r12 = np.sqrt(np.clip(s12, 1e-300, None))
    e1 = (s12 - m2 * m2 + m1 * m1) / (2 * r12)
    e3 = (M * M - s12 - m3 * m3) / (2 * r12)
    p1 = np.sqrt(np.clip(e1 * e1 - m1 * m1, 0, None))
    p3 = np.sqrt(np.clip(e3 * e3 - m3 * m3, 0, None))
    lo = (e1 + e3) ** 2 - (p1 + p3) ** 2
    hi = (e1 + e3) ** 2 - (p1 - p3) ** 2
    inside = (s12 >= (m1 + m2) ** 2) & (s12 <= (M - m3) ** 2) & (s13 >= lo) & (s13 <= hi)

    def q2(s, a, b):
        return np.clip((s - (a + b) ** 2) * (s - (a - b) ** 2) / (4 * s), 0, None)

    A = np.zeros_like(s12, dtype=np.complex128)
    for mass, width, cre, cim, ch, spin in res:
        i, j = ch // 10, ch % 10
        k = 6 - i - j
        sv = {12: s12, 13: s13, 23: s23}
        sij = sv[ch]
        sik = sv[int(f"{min(i, k)}{max(i, k)}")]
        sjk = sv[int(f"{min(j, k)}{max(j, k)}")]
        qq = q2(sij, mm[i], mm[j])
        q0 = q2(mass * mass, mm[i], mm[j])
        x = np.sqrt(qq) / np.sqrt(q0)
        if spin == 1:
            bf2 = (1 + R * R * q0) / (1 + R * R * qq)
            ratio = x ** 3
            Z = sjk - sik + (M * M - mm[k] ** 2) * (mm[i] ** 2 - mm[j] ** 2) / sij
        else:
            bf2, ratio, Z = 1.0, x, 1.0
        g = width * ratio * mass / np.sqrt(sij) * bf2
        A += complex(cre, cim) * Z * np.sqrt(bf2) / (mass * mass - sij - 1j * mass * g)
    return np.where(inside, np.abs(A) ** 2, 0.0)


class C5TI(Workload):
    name = "C5TI"
    description = ("DalitzPlotPdf D0 -> pi+ pi- pi0 (rho+, rho-, rho0, f0(980) isobars), time-integrated, "
                   "m12^2 x m13^2 grid 1024")
    default_n = 10_000_000
    fit_n = 20_000
    has_reference = False  # DalitzPlotPdf
    M, ms, R = 1.86484, (0.13957, 0.13957, 0.13498), 1.5
    # (name, channel, spin, mass, width, Re c, Im c); rho+ is the reference amplitude
    res = [("rhop", 13, 1, 0.7753, 0.1491, 1.0, 0.0),
           ("rhom", 23, 1, 0.7753, 0.1491, 0.65, 0.05),
           ("rho0", 12, 1, 0.7753, 0.1491, 0.53, 0.16),
           ("f0", 12, 0, 0.980, 0.050, 0.08, 0.12)]
    truth = {}
    start = {}
    for _n, _ch, _sp, _m, _w, _re, _im in res:
        truth.update({f"{_n}_m": _m, f"{_n}_w": _w, f"{_n}_re": _re, f"{_n}_im": _im})
        start.update({f"{_n}_m": _m, f"{_n}_w": _w * 1.02, f"{_n}_re": _re * 0.98 if _re != 1.0 else 1.0,
                      f"{_n}_im": _im + 0.01 if _n != "rhop" else 0.0})

    @classmethod
    def box(cls):
        M, (m1, m2, m3) = cls.M, cls.ms
        return ((m1 + m2) ** 2, (M - m3) ** 2), ((m1 + m3) ** 2, (M - m2) ** 2)

    def build(self, pf):
        (a12, b12), (a13, b13) = self.box()
        s12 = pf.new_observable("m12sq", a12, b12)
        s13 = pf.new_observable("m13sq", a13, b13)
        resonances = []
        for nm, ch, sp, m, w, re, im in self.res:
            mv = pf.new_parameter(f"{nm}_m", self.start[f"{nm}_m"], 0.001, m - 0.05, m + 0.05)
            wv = pf.new_parameter(f"{nm}_w", self.start[f"{nm}_w"], 0.001, 0.01, 0.5)
            cr = pf.new_parameter(f"{nm}_re", self.start[f"{nm}_re"], 0.01, -5.0, 5.0)
            ci = pf.new_parameter(f"{nm}_im", self.start[f"{nm}_im"], 0.01, -5.0, 5.0)
            mv.fixed = wv.fixed = True  # lineshapes fixed, couplings float
            if nm == "rhop":
                cr.fixed = ci.fixed = True  # the reference amplitude
            resonances.append((mv, wv, cr, ci, ch, sp))
        return [s12, s13], pf.dalitz_pdf("d0pipipi0", s12, s13, resonances, (self.M,) + self.ms, self.R)

    @classmethod
    def columns(cls, n, seed=11):
        """accept-reject with the truth couplings under a piecewise-constant
        envelope (64 x 64 cells, cell maxima from 16 x 16 sub-samples x 1.5)"""
        rng = np.random.default_rng(seed)
        (a12, b12), (a13, b13) = cls.box()
        res = [(m, w, re, im, ch, sp) for _, ch, sp, m, w, re, im in cls.res]
        nc, sub = 64, 16
        h12, h13 = (b12 - a12) / nc, (b13 - a13) / nc
        u = (np.arange(sub) + 0.5) / sub
        f12 = (a12 + (np.arange(nc)[:, None] + u[None, :]) * h12).ravel()
        f13 = (a13 + (np.arange(nc)[:, None] + u[None, :]) * h13).ravel()
        g12, g13 = np.meshgrid(f12, f13, indexing="ij")
        with np.errstate(all="ignore"):
            v = dalitz_amplitude2(g12.ravel(), g13.ravel(), cls.M, cls.ms, cls.R, res)
        env = 1.5 * v.reshape(nc, sub, nc, sub).max(axis=(1, 3)).ravel()
        env[env <= 0] = 0.0
        # cells touching the boundary: their sub-sample max may miss the plot
        p = env / env.sum()
        out = np.empty((2, n))
        filled = 0
        while filled < n:
            k = min(2 * (n - filled) + 4096, 1 << 22)
            cell = rng.choice(nc * nc, size=k, p=p)
            c12 = a12 + (cell // nc + rng.random(k)) * h12
            c13 = a13 + (cell % nc + rng.random(k)) * h13
            with np.errstate(all="ignore"):
                f = dalitz_amplitude2(c12, c13, cls.M, cls.ms, cls.R, res)
            keep = rng.random(k) * env[cell] < f
            take = min(int(keep.sum()), n - filled)
            out[0, filled:filled + take] = c12[keep][:take]
            out[1, filled:filled + take] = c13[keep][:take]
            filled += take
        return out

    def data(self, pf, obs, n, seed=11):
        return pf.UnbinnedDataSet.from_columns(obs, self.columns(n, seed))

    def bytes_per_unit(self):
        return 16.0


class C5(C5TI):
    """BASELINE config 5: the time-dependent Dalitz-plot fit (TddpPdf) of
    D0 -> pi+ pi- pi0 with the C5TI isobars, decay time t in [0, 10 tau]
    and mixing parameters x, y (pfb200.h), 1e7 events."""
    name = "C5"
    description = ("TddpPdf D0 -> pi+ pi- pi0 (rho+, rho-, rho0, f0(980) isobars) with mixing, "
                   "(m12^2, m13^2, t) grid 1024")
    tau, x_mix, y_mix = 0.4101, 0.0039, 0.0065  # ps; D0 lifetime and mixing (PDG-like)
    tmax = 10 * 0.4101
    truth = dict(C5TI.truth, tau=tau, x=x_mix, y=y_mix)
    start = dict(C5TI.start, tau=0.41, x=0.004, y=0.006)

    def build(self, pf):
        (a12, b12), (a13, b13) = self.box()
        s12 = pf.new_observable("m12sq", a12, b12)
        s13 = pf.new_observable("m13sq", a13, b13)
        t = pf.new_observable("t", 0.0, self.tmax)
        resonances = []
        for nm, ch, sp, m, w, re, im in self.res:
            mv = pf.new_parameter(f"{nm}_m", self.start[f"{nm}_m"], 0.001, m - 0.05, m + 0.05)
            wv = pf.new_parameter(f"{nm}_w", self.start[f"{nm}_w"], 0.001, 0.01, 0.5)
            cr = pf.new_parameter(f"{nm}_re", self.start[f"{nm}_re"], 0.01, -5.0, 5.0)
            ci = pf.new_parameter(f"{nm}_im", self.start[f"{nm}_im"], 0.01, -5.0, 5.0)
            mv.fixed = wv.fixed = True
            if nm == "rhop":
                cr.fixed = ci.fixed = True
            resonances.append((mv, wv, cr, ci, ch, sp))
        tau = pf.new_parameter("tau", self.start["tau"], 0.001, 0.2, 0.8)
        x = pf.new_parameter("x", self.start["x"], 0.001, -0.2, 0.2)
        y = pf.new_parameter("y", self.start["y"], 0.001, -0.2, 0.2)
        return [s12, s13, t], pf.tddp_pdf("d0tddp", s12, s13, t, resonances, (self.M,) + self.ms, tau, x, y, self.R)

    @classmethod
    def columns(cls, n, seed=11):
        """accept-reject under (|A|^2 + |Abar|^2) e^-((1 - |y|) t / tau), which
        bounds |A g+ + Abar g-|^2 (Cauchy-Schwarz; e^-T cosh yT <= e^-(1-|y|)T):
        cell envelope of (|A|^2 + |Abar|^2) as C5TI's, t from the truncated
        exponential of lifetime tau / (1 - |y|)"""
        rng = np.random.default_rng(seed)
        (a12, b12), (a13, b13) = cls.box()
        res = [(m, w, re, im, ch, sp) for _, ch, sp, m, w, re, im in cls.res]
        M, ms = cls.M, cls.ms
        msum = M * M + sum(v * v for v in ms)

        def both(c12, c13):
            c23 = msum - c12 - c13
            A = dalitz_amplitude(c12, c13, c23, M, ms, cls.R, res)
            Ab = dalitz_amplitude(c12, c23, c13, M, ms, cls.R, res)
            return np.where(dalitz_inside(c12, c13, M, ms), np.abs(A) ** 2 + np.abs(Ab) ** 2, 0.0)

        nc, sub = 64, 16
        h12, h13 = (b12 - a12) / nc, (b13 - a13) / nc
        u = (np.arange(sub) + 0.5) / sub
        f12 = (a12 + (np.arange(nc)[:, None] + u[None, :]) * h12).ravel()
        f13 = (a13 + (np.arange(nc)[:, None] + u[None, :]) * h13).ravel()
        g12, g13 = np.meshgrid(f12, f13, indexing="ij")
        with np.errstate(all="ignore"):
            v = both(g12.ravel(), g13.ravel())
        env = 1.5 * v.reshape(nc, sub, nc, sub).max(axis=(1, 3)).ravel()
        env[env <= 0] = 0.0
        p = env / env.sum()
        rate = (1.0 - abs(cls.y_mix)) / cls.tau
        cut = 1.0 - np.exp(-rate * cls.tmax)
        out = np.empty((3, n))
        filled = 0
        while filled < n:
            k = min(2 * (n - filled) + 4096, 1 << 21)
            cell = rng.choice(nc * nc, size=k, p=p)
            c12 = a12 + (cell // nc + rng.random(k)) * h12
            c13 = a13 + (cell % nc + rng.random(k)) * h13
            ct = -np.log1p(-rng.random(k) * cut) / rate
            with np.errstate(all="ignore"):
                f = tddp_density(c12, c13, ct, M, ms, cls.R, res, cls.tau, cls.x_mix, cls.y_mix)
            keep = rng.random(k) * env[cell] * np.exp(-rate * ct) < f
            take = min(int(keep.sum()), n - filled)
            out[0, filled:filled + take] = c12[keep][:take]
            out[1, filled:filled + take] = c13[keep][:take]
            out[2, filled:filled + take] = ct[keep][:take]
            filled += take
        return out

    def bytes_per_unit(self):
        return 24.0


WORKLOADS = {w.name: w for w in (C1(), C2(), C3(), C4(), C5(), C5TI())}
