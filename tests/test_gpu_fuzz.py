"""Randomised parity: seeded random PDF trees (Exp, Gauss, Breit-Wigner,
Polynomial, Argus, AddPdf, ProdPdf, Mapped, Convolution; Composite and
Dalitz are covered by the golden and C5 tests) on one or two observables, evaluated through the C ABI and by
the C oracle at several parameter points.  Exercises the code generator's
combinations that the golden cases do not: folded AddPdf / ProdPdf norms
at several levels, both log-domain forms and their fast paths, mixtures of
log-linear and linear children, nested combinators.  Bar: NLL within 1e-12
relative and the root norm within 1e-12."""
import numpy as np
import pytest

import oracle
from paper_1311_1753_b200 import parfit as pf

pytestmark = pytest.mark.gpu
REL = 1e-12


class _Builder:
    def __init__(self, rng, obs):
        self.rng = rng
        self.obs = obs
        self.n = 0
        self.defs = []  # (variable, sampler of valid values)

    def par(self, lo, hi, init=None):
        self.n += 1
        v = pf.new_parameter(f"p{self.n}", init if init is not None else self.rng.uniform(lo, hi), 0.01, lo, hi)
        self.defs.append((v, lo, hi))
        return v

    def name(self, k):
        self.n += 1
        return f"{k}{self.n}"

    def leaf(self, x, allow=("exp", "gauss", "bw", "poly")):
        k = self.rng.choice(allow)
        lo, hi = x.lower, x.upper
        if k == "exp":
            return pf.exp_pdf(self.name("e"), x, self.par(-1.0, 0.5))
        if k == "gauss":
            return pf.gaussian_pdf(self.name("g"), x, self.par(lo, hi), self.par(0.2 * (hi - lo), 0.6 * (hi - lo)))
        if k == "bw":
            return pf.breit_wigner_pdf(self.name("b"), x, self.par(lo + 0.2 * (hi - lo), hi - 0.2 * (hi - lo)),
                                       self.par(0.1 * (hi - lo), 0.5 * (hi - lo)))
        return pf.polynomial_pdf(self.name("q"), x, [self.par(0.5, 2.0), self.par(-0.1, 0.1), self.par(0.0, 0.02)])

    def tree(self, depth, root=False):
        x, y = self.obs
        r = self.rng.uniform(0.3, 1.0) if root else self.rng.random()
        if depth == 0 or r < 0.3:
            return self.leaf(x)
        if r < 0.55:  # mixture of 2-3 children on x
            k = int(self.rng.integers(2, 4))
            ch = [self.tree(depth - 1) for _ in range(k)]
            fr = [self.par(0.05, 0.9 / (k - 1)) for _ in range(k - 1)]
            return pf.add_pdf(self.name("a"), ch, fr)
        if r < 0.75:  # separable product with a y factor (Argus or exp/gauss)
            fy = (pf.argus_pdf(self.name("r"), y, self.par(y.upper + 0.001, y.upper + 0.01), self.par(-30, -1),
                               self.par(0.3, 1.5))
                  if self.rng.random() < 0.5 else self.leaf(y, ("exp", "gauss")))
            return pf.prod_pdf(self.name("p"), [self.tree(depth - 1), fy])
        if r < 0.85:  # product on the same observable (not separable)
            return pf.prod_pdf(self.name("p"), [self.leaf(x, ("exp", "gauss")), self.leaf(x, ("gauss", "poly"))])
        if r < 0.93:  # mapped over two halves of x
            mid = 0.5 * (x.lower + x.upper)
            return pf.mapped_pdf(self.name("m"), [x.lower, mid, x.upper], [self.leaf(x), self.leaf(x)])
        # convolution: steep models (|alpha| sigma up to ~5, the regime where a
        # fixed resolution window would drop the dominant terms) and
        # polynomials that clamp inside the quadrature table
        k = self.rng.choice(("steep", "bw", "poly"))
        lo, hi = x.lower, x.upper
        if k == "steep":
            model = pf.exp_pdf(self.name("e"), x, self.par(-12.0, 6.0))
        elif k == "poly":
            model = pf.polynomial_pdf(self.name("q"), x, [self.par(-0.5, 1.5), self.par(-0.6, 0.3)])
        else:
            model = self.leaf(x, ("bw",))
        return pf.convolution_pdf(self.name("c"), model,
                                  pf.gaussian_pdf(self.name("g"), x, self.par(-0.05, 0.05, 0.0),
                                                  self.par(0.05, 0.4)), int(self.rng.choice([32, 256])))

    def point(self, order):
        lookup = {v.name: (lo, hi) for v, lo, hi in self.defs}
        out = []
        for nm in order:
            lo, hi = lookup[nm]
            out.append(self.rng.uniform(lo, hi))
        return out


@pytest.mark.parametrize("seed", range(40))
def test_random_model_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    x = pf.new_observable("x", 0.0, 4.0)
    y = pf.new_observable("y", 5.20, 5.29)
    b = _Builder(rng, (x, y))
    pdf = b.tree(3, root=True)
    n = int(rng.integers(1, 3000))
    cols = np.stack([4.0 * rng.random(n), 5.20 + 0.09 * rng.random(n)])
    ds = pf.UnbinnedDataSet.from_columns([x, y], cols)
    grid = 64
    try:
        want_model = oracle.Oracle(pdf, ds, grid)
    except oracle.OracleError as e:  # a contract the oracle refuses must be refused on the GPU too
        with pytest.raises(pf.Error):
            pf.BoundModel(pdf, ds, pf.GridSpec(grid))
        pytest.skip(f"model refused consistently: {e}")
    bm = pf.BoundModel(pdf, ds, pf.GridSpec(grid))
    names = [v.name for v in bm.registry().parameters()]
    assert names == want_model.param_names()
    nodes = pf.GraphDesc(pdf, [x, y]).preorder()
    for _ in range(3):
        p = b.point(names)
        try:
            want = want_model.eval(p)
        except oracle.OracleError as e:
            with pytest.raises(pf.Error) as ei:
                bm.eval_metric(p)
            assert ei.value.args[0].split(":")[0] == str(e).split(":")[0]
            continue
        got = bm.eval_metric(p)
        assert abs(got - want) <= REL * max(abs(want), 1.0), (seed, p, got, want)
        if want != pf.kPenaltyValue:
            norms, _, valid = want_model.norms()
            if valid[0]:
                assert abs(nodes[0].cached_norm() - norms[0]) <= REL * abs(norms[0]), (seed, p)
        assert bm.log_floor_count() == want_model.floor_count()
        for i, nd in enumerate(nodes):  # PolynomialPdf clamps, per raw call (pdf.hpp:313-316)
            if isinstance(nd, pf.PolynomialPdf):
                assert nd.clamp_count() == want_model.clamp_count(i), (seed, nd.name)
