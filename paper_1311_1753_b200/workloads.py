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


WORKLOADS = {w.name: w for w in (C1(), C2(), C3(), C4())}
