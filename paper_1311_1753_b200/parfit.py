"""Python mirror of the reference ``parfit`` API over the B200 engine.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/parfit/*.hpp, cited per class), so a test
written against the reference reads the same here.  All metric work runs in
libpfb200.so on the GPU (include/pfb200.h); this module only describes the
graph and the data, and marshals calls.

Drop-in map: GooFit ``Variable`` -> :func:`new_observable` /
:func:`new_parameter`; ``GooPdf`` -> :class:`PdfNode`; ``setData`` ->
:class:`BoundModel`; ``FitManager`` -> :func:`fit` (and :class:`FitManager`).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import lib


class Error(RuntimeError):
    """parfit::Error (errors.hpp:11-16): message "code: detail"."""

    def __init__(self, code_or_msg: str, detail: Optional[str] = None):
        msg = code_or_msg if detail is None else f"{code_or_msg}: {detail}"
        super().__init__(msg)
        self.code = msg.split(":", 1)[0]


def _raise(st: _abi.pf_status):
    raise Error(st.message.decode())


# ---------------------------------------------------------------------------
# variable.hpp

class Role(enum.IntEnum):
    Observable = _abi.PF_OBSERVABLE
    Parameter = _abi.PF_PARAMETER


class Variable:
    """parfit::Variable (variable.hpp:18-27).  Identity matters."""

    __slots__ = ("name", "value", "lower", "upper", "step", "fixed", "role", "global_index")

    def __init__(self, name, value, lower, upper, step, role):
        self.name = name
        self.value = float(value)
        self.lower = float(lower)
        self.upper = float(upper)
        self.step = float(step)
        self.fixed = False
        self.role = role
        self.global_index = -1

    def __repr__(self):
        return f"Variable({self.name!r}, value={self.value}, [{self.lower}, {self.upper}])"


def new_observable(name: str, lower: float, upper: float) -> Variable:
    """variable.hpp:31-42"""
    if not (lower < upper):
        raise Error("invalid-range", f"observable '{name}': lower must be < upper")
    return Variable(name, lower, lower, upper, 0.0, Role.Observable)


def new_parameter(name: str, init: float, step: float, lower: float, upper: float) -> Variable:
    """variable.hpp:44-60"""
    if not (lower < upper):
        raise Error("invalid-range", f"parameter '{name}': lower must be < upper")
    if not (lower <= init <= upper):
        raise Error("invalid-range", f"parameter '{name}': init outside [lower, upper]")
    if not (step > 0):
        raise Error("invalid-step", f"parameter '{name}': step must be > 0")
    return Variable(name, init, lower, upper, step, Role.Parameter)


class ParameterRegistry:
    """variable.hpp:65-121: registration order is the parameter-vector layout."""

    def __init__(self):
        self._params: List[Variable] = []
        self._obs: List[Variable] = []
        self._pby: dict = {}
        self._oby: dict = {}

    def _register(self, lst, by, v):
        have = by.get(v.name)
        if have is not None:
            if have is not v:
                raise Error("name-collision", f"distinct Variables both named '{v.name}'")
            return have.global_index
        v.global_index = len(lst)
        lst.append(v)
        by[v.name] = v
        return v.global_index

    def register_parameter(self, v: Variable) -> int:
        if v is None:
            raise Error("null-variable", "register_parameter")
        if v.role != Role.Parameter:
            raise Error("wrong-role", f"'{v.name}' is not a parameter")
        return self._register(self._params, self._pby, v)

    def register_observable(self, v: Variable) -> int:
        if v is None:
            raise Error("null-variable", "register_observable")
        if v.role != Role.Observable:
            raise Error("wrong-role", f"'{v.name}' is not an observable")
        return self._register(self._obs, self._oby, v)

    def parameters(self) -> List[Variable]:
        return list(self._params)

    def observables(self) -> List[Variable]:
        return list(self._obs)

    def n_parameters(self) -> int:
        return len(self._params)

    def export_values(self) -> List[float]:
        return [p.value for p in self._params]

    def import_values(self, vals: Sequence[float]):
        if len(vals) != len(self._params):
            raise Error("size-mismatch", "import_values: wrong parameter count")
        for p, v in zip(self._params, vals):
            p.value = float(v)


# ---------------------------------------------------------------------------
# dataset.hpp

class UnbinnedDataSet:
    """dataset.hpp:20-51.  add_event() snapshots the observables' values;
    from_columns() binds a whole column-major block at once."""

    def __init__(self, observables):
        if isinstance(observables, Variable):
            observables = [observables]
        observables = list(observables)
        if not observables:
            raise Error("empty-observables", "UnbinnedDataSet needs >= 1 observable")
        for i in range(len(observables)):
            for j in range(i + 1, len(observables)):
                if observables[i] is observables[j] or observables[i].name == observables[j].name:
                    raise Error("duplicate-observable", observables[i].name)
        self._obs = observables
        self._rows: list = []
        self._block = np.zeros((len(observables), 0))

    @classmethod
    def from_columns(cls, observables, columns) -> "UnbinnedDataSet":
        ds = cls(observables)
        arr = np.ascontiguousarray(np.asarray(columns, dtype=np.float64).reshape(len(ds._obs), -1))
        ds._block = arr
        return ds

    def add_event(self):
        self._rows.append(tuple(o.value for o in self._obs))

    def _consolidate(self):
        if self._rows:
            extra = np.asarray(self._rows, dtype=np.float64).T.reshape(len(self._obs), -1)
            self._block = np.ascontiguousarray(np.concatenate([self._block, extra], axis=1))
            self._rows = []
        return self._block

    def observables(self):
        return list(self._obs)

    def columns(self) -> np.ndarray:
        """column-major EventTable values, shape (n_columns, n_events)"""
        return self._consolidate()

    def rows(self):
        return [list(r) for r in self._consolidate().T]

    def n_events(self) -> int:
        return self._block.shape[1] + len(self._rows)

    def n_columns(self) -> int:
        return len(self._obs)


# ---- event-store I/O --------------------------------------------------------
def write_text(ds: UnbinnedDataSet, out) -> None:
    """dataset.hpp:187-200: '#' header naming the observables, then one event
    per line, columns in observable order, %.17g (round-trip precision)"""
    cols = ds.columns()
    out.write("#" + "".join(" " + o.name for o in ds.observables()) + "\n")
    if cols.shape[1]:
        np.savetxt(out, cols.T, fmt="%.17g", delimiter=" ")


def write_text_file(ds: UnbinnedDataSet, path: str) -> None:
    try:
        fh = open(path, "w")
    except OSError:
        raise Error("io-error", f"cannot open '{path}' for writing") from None
    with fh:
        write_text(ds, fh)


def read_text(inp, observables) -> UnbinnedDataSet:
    """dataset.hpp:208-238 (same header check and error codes)"""
    observables = list(observables)
    header = inp.readline()
    if not header or not header.startswith("#"):
        raise Error("bad-format", "missing '#' header line")
    names = header[1:].split()
    for i, name in enumerate(names):
        if i >= len(observables) or observables[i].name != name:
            raise Error("bad-format", f"header observable '{name}' does not match expected order")
    if len(names) != len(observables):
        raise Error("bad-format", "header names fewer observables than expected")
    rows = []
    for line in inp:
        parts = line.split()
        if not parts:
            continue
        if len(parts) < len(observables):
            raise Error("bad-format", "short row in data file")
        try:
            rows.append([float(v) for v in parts[:len(observables)]])
        except ValueError:
            raise Error("bad-format", "short row in data file") from None
    cols = np.asarray(rows, dtype=np.float64).reshape(-1, len(observables)).T
    return UnbinnedDataSet.from_columns(observables, cols)


def read_text_file(path: str, observables) -> UnbinnedDataSet:
    try:
        fh = open(path)
    except OSError:
        raise Error("io-error", f"cannot open '{path}'") from None
    with fh:
        return read_text(fh, observables)


_BIN_MAGIC = b"PFB200EV"


def write_binary_file(ds: UnbinnedDataSet, path: str) -> None:
    """binary event store for large fixtures: magic, n_obs, n_events (uint64),
    the observable names (NUL-separated), then the column-major float64
    EventTable as it lies in HBM"""
    cols = np.ascontiguousarray(ds.columns(), dtype="<f8")
    names = b"\0".join(o.name.encode() for o in ds.observables())
    with open(path, "wb") as fh:
        fh.write(_BIN_MAGIC)
        fh.write(np.array([cols.shape[0], cols.shape[1], len(names)], dtype="<u8").tobytes())
        fh.write(names)
        fh.write(cols.tobytes())


def read_binary_file(path: str, observables) -> UnbinnedDataSet:
    observables = list(observables)
    try:
        fh = open(path, "rb")
    except OSError:
        raise Error("io-error", f"cannot open '{path}'") from None
    with fh:
        if fh.read(8) != _BIN_MAGIC:
            raise Error("bad-format", "not a pfb200 binary event store")
        n_obs, n_ev, nlen = (int(v) for v in np.frombuffer(fh.read(24), dtype="<u8"))
        names = fh.read(nlen).split(b"\0") if nlen else []
        if [n.decode() for n in names] != [o.name for o in observables] or n_obs != len(observables):
            raise Error("bad-format", "observables do not match the file's")
        cols = np.frombuffer(fh.read(8 * n_obs * n_ev), dtype="<f8")
        if cols.size != n_obs * n_ev:
            raise Error("bad-format", "truncated event store")
    return UnbinnedDataSet.from_columns(observables, cols.reshape(n_obs, n_ev))


# ---- toy generation (generate.hpp) -------------------------------------------
class ToyRng:
    """generate.hpp:19-27: uniforms (mt19937_64() >> 11) * 2^-53 from a fixed
    bit recipe, so identical seeds give identical samples everywhere.  Host
    side (a plain mt19937_64); generate_events draws the same stream on the
    GPU."""

    _N, _M = 312, 156

    def __init__(self, seed: int):
        m = [0] * self._N
        m[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self._N):
            m[i] = (6364136223846793005 * (m[i - 1] ^ (m[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self._mt, self._i = m, self._N

    def _twist(self):
        m, N, M = self._mt, self._N, self._M
        for i in range(N):
            y = (m[i] & 0xFFFFFFFF80000000) | (m[(i + 1) % N] & 0x7FFFFFFF)
            m[i] = m[(i + M) % N] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
        self._i = 0

    def next_u64(self) -> int:
        if self._i >= self._N:
            self._twist()
        y = self._mt[self._i]
        self._i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def uniform(self, lo: Optional[float] = None, hi: Optional[float] = None) -> float:
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u


def generate_events(pdf: "PdfNode", observables, n_events: int, seed: int,
                    grid: Optional["GridSpec"] = None, device: int = 0) -> UnbinnedDataSet:
    """generate_events (generate.hpp:33-86) on the GPU: the reference's
    envelope, ToyRng stream and accept-reject order, so a seed gives the
    reference's sample.  Sets each box observable's value to the last
    accepted event, as the reference does."""
    grid = grid or GridSpec()
    observables = list(observables)
    g = GraphDesc(pdf, observables)
    idx = (C.c_int32 * max(len(observables), 1))(*[g.var_index(o) for o in observables])
    n = int(n_events)
    out = np.empty((len(observables), max(n, 1)))
    last = (C.c_double * max(len(observables), 1))()
    ms = C.c_double()
    opt = _abi.pf_options(device, 1, 0, 1, 0)
    st = _abi.pf_status()
    if lib.pf_generate_events(C.byref(g.c_graph), idx, len(observables), max(n, 0), seed & 0xFFFFFFFFFFFFFFFF,
                              grid.points, C.byref(opt), out.ctypes.data_as(C.POINTER(C.c_double)), last,
                              C.byref(ms), C.byref(st)):
        _raise(st)
    for i, o in enumerate(observables):
        o.value = last[i]
    ds = UnbinnedDataSet.from_columns(observables, out)
    ds.generation_ms = ms.value
    return ds


class BinnedDataSet:
    """dataset.hpp:55-129: uniform bins, last upper edge inclusive."""

    def __init__(self, observables, bins):
        observables = list(observables)
        bins = [int(b) for b in bins]
        if not observables:
            raise Error("empty-observables", "BinnedDataSet needs >= 1 observable")
        if len(observables) != len(bins):
            raise Error("dimension-mismatch", "observable/bin count mismatch")
        if any(b < 1 for b in bins):
            raise Error("dimension-mismatch", "bins must be >= 1")
        self._obs = observables
        self._bins = bins
        self._contents = np.zeros(int(np.prod(bins)), dtype=np.float64)

    def flat_bin(self, point) -> int:
        idx = 0
        for i, o in enumerate(self._obs):
            w = (o.upper - o.lower) / float(self._bins[i])
            x = float(point[i])
            if x < o.lower or x > o.upper:
                raise Error("out-of-range", f"fill: '{o.name}' outside range")
            b = int((x - o.lower) / w)
            if b >= self._bins[i]:
                if x == o.upper:
                    b = self._bins[i] - 1
                else:
                    raise Error("out-of-range", f"fill: '{o.name}' outside range")
            if x == o.upper and b != self._bins[i] - 1:
                raise Error("out-of-range", f"fill: '{o.name}' at excluded edge")
            idx = idx * self._bins[i] + b
        return idx

    def fill(self, point, weight: float = 1.0):
        if len(point) != len(self._obs):
            raise Error("dimension-mismatch", "fill point arity")
        self._contents[self.flat_bin(point)] += weight

    def set_contents(self, contents):
        c = np.asarray(contents, dtype=np.float64).ravel()
        if c.size != self._contents.size:
            raise Error("dimension-mismatch", "contents size")
        self._contents = c.copy()

    def bin_center(self, obs: int, b: int) -> float:
        o = self._obs[obs]
        w = (o.upper - o.lower) / float(self._bins[obs])
        return o.lower + (float(b) + 0.5) * w

    def bin_volume(self) -> float:
        v = 1.0
        for i, o in enumerate(self._obs):
            v *= (o.upper - o.lower) / float(self._bins[i])
        return v

    def total_content(self) -> float:
        # std::accumulate: sequential double sum (dataset.hpp:356-358)
        if self._contents.size == 0:
            return 0.0
        return float(np.add.accumulate(self._contents)[-1])

    def observables(self):
        return list(self._obs)

    def bins(self):
        return list(self._bins)

    def contents(self):
        return self._contents

    def n_bins(self) -> int:
        return int(self._contents.size)


def to_event_table(ds) -> np.ndarray:
    """dataset.hpp:150-182: column-major values (n_columns, n_events)."""
    if isinstance(ds, UnbinnedDataSet):
        return ds.columns()
    nobs = len(ds.observables())
    n = ds.n_bins()
    out = np.empty((nobs + 2, n))
    flat = np.arange(n)
    rem = flat.copy()
    idx = [None] * nobs
    for i in range(nobs - 1, -1, -1):
        idx[i] = rem % ds.bins()[i]
        rem //= ds.bins()[i]
    for i, o in enumerate(ds.observables()):
        w = (o.upper - o.lower) / float(ds.bins()[i])
        out[i] = o.lower + (idx[i].astype(np.float64) + 0.5) * w
    out[nobs] = ds.contents()
    out[nobs + 1] = ds.bin_volume()
    return out


# ---------------------------------------------------------------------------
# pdf.hpp

class GridSpec:
    """pdf.hpp:32-38"""

    def __init__(self, points: int = 1024):
        if points < 2:
            raise Error("bad-grid", "GridSpec needs >= 2 points")
        self.points = int(points)


class PdfNode:
    """PdfNode (pdf.hpp:61-205).  raw() kernels live on the GPU; after an
    evaluation the node exposes the cached norm the device computed."""

    kind = -1

    def __init__(self, name: str):
        self._name = name
        self._children: List["PdfNode"] = []
        self._params: List[Variable] = []
        self._obs: List[Variable] = []
        self._reals: List[float] = []
        self._q = 0
        self._id = 0
        self._norm = 1.0
        self._norm_err = 0.0
        self._norm_valid = False
        self._owner = None  # the BoundModel that evaluated this node last (norms fetched lazily)
        self._model = None

    def name(self):
        return self._name

    def id(self):
        return self._id

    def children(self):
        return list(self._children)

    def declared_parameters(self):
        return list(self._params)

    def declared_observables(self):
        return list(self._obs)

    def _fresh(self):
        if self._owner is not None and self._owner._stale:
            self._owner._sync_norms()

    def cached_norm(self) -> float:
        self._fresh()
        if not self._norm_valid:
            raise Error("stale-normalization", self._name)
        return self._norm

    def norm_error_estimate(self) -> float:
        self._fresh()
        return self._norm_err


def _need_obs(name, v, what="x"):
    if v is None or v.role != Role.Observable:
        raise Error("wrong-role", f"{name}: {what} must be an observable")


def _need_par(name, v, what):
    if v is None or v.role != Role.Parameter:
        raise Error("wrong-role", f"{name}: {what} must be a parameter")


class ExpPdf(PdfNode):
    kind = _abi.PF_EXPONENTIAL

    def __init__(self, name, x, alpha):  # pdf.hpp:212-217
        super().__init__(name)
        _need_obs(name, x)
        _need_par(name, alpha, "alpha")
        self._obs = [x]
        self._params = [alpha]


class GaussianPdf(PdfNode):
    kind = _abi.PF_GAUSSIAN

    def __init__(self, name, x, mean, sigma):  # pdf.hpp:237-249
        super().__init__(name)
        _need_obs(name, x)
        _need_par(name, mean, "mean")
        _need_par(name, sigma, "sigma")
        if not (sigma.lower > 0):
            raise Error("nonpositive-sigma", f"{name}: sigma limits must exclude 0")
        self._obs = [x]
        self._params = [mean, sigma]


class BreitWignerPdf(PdfNode):
    kind = _abi.PF_BREIT_WIGNER

    def __init__(self, name, x, mass, width):  # pdf.hpp:266-278
        super().__init__(name)
        _need_obs(name, x)
        _need_par(name, mass, "mass")
        _need_par(name, width, "width")
        if not (width.lower > 0):
            raise Error("nonpositive-width", f"{name}: width limits must exclude 0")
        self._obs = [x]
        self._params = [mass, width]


class PolynomialPdf(PdfNode):
    kind = _abi.PF_POLYNOMIAL

    def __init__(self, name, x, coeffs):  # pdf.hpp:294-305
        super().__init__(name)
        _need_obs(name, x)
        coeffs = list(coeffs)
        if not coeffs:
            raise Error("bad-arity", f"{name}: need >= 1 coefficient")
        for c in coeffs:
            if c is None or c.role != Role.Parameter:
                raise Error("wrong-role", f"{name}: coefficients must be parameters")
        self._obs = [x]
        self._params = coeffs

    def clamp_count(self) -> int:
        if self._model is None:
            return 0
        return int(lib.pf_clamp_count(self._model._h, self._id))


class ArgusPdf(PdfNode):
    """ArgusPdf(x; m0, c, p) = x (1 - (x/m0)^2)^p exp(c (1 - (x/m0)^2)) for
    x < m0, else 0 (GooFit's upper-threshold form).  Not in the reference;
    needed by BASELINE config 3."""

    kind = _abi.PF_ARGUS

    def __init__(self, name, x, m0, c, p):
        super().__init__(name)
        _need_obs(name, x)
        for v, w in ((m0, "m0"), (c, "c"), (p, "p")):
            _need_par(name, v, w)
        if not (m0.lower > 0):
            raise Error("nonpositive-endpoint", f"{name}: m0 limits must exclude 0")
        self._obs = [x]
        self._params = [m0, c, p]


class DalitzPlotPdf(PdfNode):
    """Time-integrated isobar model over the Dalitz plot of M -> 1 2 3:
    |sum_r c_r BW_r|^2 inside the kinematic boundary, 0 outside.
    Observables m12^2, m13^2.  Each resonance is (mass, width, Re c, Im c)
    parameters plus a channel (12, 13 or 23) and spin (0 or 1); BW_r is a
    relativistic Breit-Wigner with mass-dependent width, Blatt-Weisskopf
    barrier (radius R) and Zemach spin factor (pf_device.cuh / pf_oracle.c).
    Not in the reference; BASELINE config 5's amplitude part."""

    kind = _abi.PF_DALITZ

    def __init__(self, name, m12sq, m13sq, resonances, masses, radius=1.5):
        super().__init__(name)
        _need_obs(name, m12sq, "m12sq")
        _need_obs(name, m13sq, "m13sq")
        M, m1, m2, m3 = (float(v) for v in masses)
        if not (M > m1 + m2 + m3 and min(m1, m2, m3) >= 0 and radius >= 0):
            raise Error("bad-kinematics", f"{name}: need M > m1 + m2 + m3, masses and R >= 0")
        if not resonances:
            raise Error("bad-arity", f"{name}: need >= 1 resonance")
        params, reals = [], [M, m1, m2, m3, float(radius)]
        for res in resonances:
            mass, width, cre, cim, channel, spin = res
            for v, w in ((mass, "mass"), (width, "width"), (cre, "Re c"), (cim, "Im c")):
                _need_par(name, v, w)
            if channel not in (12, 13, 23):
                raise Error("bad-channel", f"{name}: channel must be 12, 13 or 23")
            if spin not in (0, 1):
                raise Error("bad-spin", f"{name}: spin must be 0 or 1")
            if not (width.lower > 0):
                raise Error("nonpositive-width", f"{name}: width limits must exclude 0")
            params += [mass, width, cre, cim]
            reals += [float(channel), float(spin)]
        self._obs = [m12sq, m13sq]
        self._params = params
        self._reals = reals


class TddpPdf(DalitzPlotPdf):
    """Time-dependent Dalitz-plot PDF of D0 -> 1 2 3 with mixing (BASELINE
    config 5; GooFit's TddpPdf of PAPER.md:299-309, restated -- not in the
    reference).  Observables m12^2, m13^2, t; the DalitzPlotPdf resonances,
    then lifetime tau and mixing parameters x, y.  With A the isobar
    amplitude and Abar(s12, s13) = A(s12, s23) its CP mirror (daughters 1 and
    2 conjugate, m1 == m2), the density is |A g+(t) + Abar g-(t)|^2:
      e^-(t/tau) [(|A|^2+|Abar|^2)/2 cosh(y t/tau) + (|A|^2-|Abar|^2)/2 cos(x t/tau)
                  - Re(A* Abar) sinh(y t/tau) - Im(A* Abar) sin(x t/tau)]
    inside the kinematic boundary, 0 outside (pfb200.h, pf_oracle.c)."""

    kind = _abi.PF_TDDP

    def __init__(self, name, m12sq, m13sq, t, resonances, masses, tau, x, y, radius=1.5):
        super().__init__(name, m12sq, m13sq, resonances, masses, radius)
        _need_obs(name, t, "t")
        for v, w in ((tau, "tau"), (x, "x"), (y, "y")):
            _need_par(name, v, w)
        if not (tau.lower > 0):
            raise Error("nonpositive-lifetime", f"{name}: tau limits must exclude 0")
        M, m1, m2, m3 = (float(v) for v in masses)
        if m1 != m2:
            raise Error("bad-kinematics", f"{name}: daughters 1 and 2 must be CP conjugates (m1 == m2)")
        self._obs = [m12sq, m13sq, t]
        self._params = self._params + [tau, x, y]


class ProdPdf(PdfNode):
    kind = _abi.PF_PRODUCT

    def __init__(self, name, children):  # pdf.hpp:332-337
        super().__init__(name)
        children = list(children)
        if len(children) < 2:
            raise Error("bad-arity", f"{name}: product needs >= 2 children")
        self._children = children


class AddPdf(PdfNode):
    kind = _abi.PF_SUM

    def __init__(self, name, children, fractions):  # pdf.hpp:354-366
        super().__init__(name)
        children, fractions = list(children), list(fractions)
        if len(children) < 2:
            raise Error("bad-arity", f"{name}: sum needs >= 2 children")
        if len(fractions) != len(children) - 1:
            raise Error("fraction-count-mismatch", f"{name}: need n_children - 1 fractions")
        for f in fractions:
            if f is None or f.role != Role.Parameter:
                raise Error("wrong-role", f"{name}: fractions must be parameters")
        self._children = children
        self._params = fractions


class CompositePdf(PdfNode):
    kind = _abi.PF_COMPOSITE

    def __init__(self, name, outer, inner):  # pdf.hpp:397-401
        super().__init__(name)
        if outer is None or inner is None:
            raise Error("bad-arity", f"{name}: null child")
        self._children = [outer, inner]


class MappedPdf(PdfNode):
    kind = _abi.PF_MAPPED

    def __init__(self, name, boundaries, targets):  # pdf.hpp:422-432
        super().__init__(name)
        boundaries, targets = [float(b) for b in boundaries], list(targets)
        if not targets:
            raise Error("bad-arity", f"{name}: need >= 1 target")
        if len(boundaries) != len(targets) + 1:
            raise Error("bad-arity", f"{name}: need n_targets + 1 boundaries")
        for i in range(1, len(boundaries)):
            if not (boundaries[i - 1] < boundaries[i]):
                raise Error("non-monotone-boundaries", name)
        self._children = targets
        self._reals = boundaries

    def boundaries(self):
        return list(self._reals)


class ConvolutionPdf(PdfNode):
    kind = _abi.PF_CONVOLUTION

    def __init__(self, name, model, resolution, quadrature_points: int = 1024):  # pdf.hpp:464-470
        super().__init__(name)
        if model is None or resolution is None:
            raise Error("bad-arity", f"{name}: null child")
        if quadrature_points < 2:
            raise Error("bad-grid", f"{name}: need >= 2 quadrature points")
        self._children = [model, resolution]
        self._q = int(quadrature_points)

    def quadrature_points(self):
        return self._q


# factories (pdf.hpp:622-660)
def exp_pdf(name, x, alpha):
    return ExpPdf(name, x, alpha)


def gaussian_pdf(name, x, mean, sigma):
    return GaussianPdf(name, x, mean, sigma)


def breit_wigner_pdf(name, x, mass, width):
    return BreitWignerPdf(name, x, mass, width)


def polynomial_pdf(name, x, coeffs):
    return PolynomialPdf(name, x, coeffs)


def dalitz_pdf(name, m12sq, m13sq, resonances, masses, radius=1.5):
    """resonances: [(mass, width, Re c, Im c, channel, spin), ...]"""
    return DalitzPlotPdf(name, m12sq, m13sq, resonances, masses, radius)


def tddp_pdf(name, m12sq, m13sq, t, resonances, masses, tau, x, y, radius=1.5):
    """resonances as dalitz_pdf; tau, x, y: lifetime and mixing parameters"""
    return TddpPdf(name, m12sq, m13sq, t, resonances, masses, tau, x, y, radius)


def argus_pdf(name, x, m0, c, p):
    return ArgusPdf(name, x, m0, c, p)


def prod_pdf(name, children):
    return ProdPdf(name, children)


def add_pdf(name, children, fractions):
    return AddPdf(name, children, fractions)


def composite_pdf(name, outer, inner):
    return CompositePdf(name, outer, inner)


def mapped_pdf(name, boundaries, targets):
    return MappedPdf(name, boundaries, targets)


def convolution_pdf(name, model, resolution, quadrature_points: int = 1024):
    return ConvolutionPdf(name, model, resolution, quadrature_points)


# ---------------------------------------------------------------------------
# graph description for the C ABI

class GraphDesc:
    """Serialises a PdfNode tree (by object identity) into pf_graph."""

    def __init__(self, root: Optional[PdfNode], data_observables: Sequence[Variable]):
        self.vars: List[Variable] = []
        self._vidx: dict = {}
        self.nodes: List[PdfNode] = []
        self._nidx: dict = {}
        for o in data_observables:
            self.var_index(o)
        self.root = self._add(root) if root is not None else -1
        self._build()

    def var_index(self, v: Variable) -> int:
        k = id(v)
        if k not in self._vidx:
            self._vidx[k] = len(self.vars)
            self.vars.append(v)
        return self._vidx[k]

    def _add(self, node: PdfNode) -> int:
        k = id(node)
        if k in self._nidx:
            return self._nidx[k]
        idx = len(self.nodes)
        self._nidx[k] = idx
        self.nodes.append(node)
        node._desc_children = [self._add(c) for c in node._children]
        node._desc_params = [self.var_index(p) for p in node._params]
        node._desc_obs = [self.var_index(o) for o in node._obs]
        return idx

    def _build(self):
        self._names = [v.name.encode() for v in self.vars]
        self.c_vars = (_abi.pf_variable * max(len(self.vars), 1))()
        for i, v in enumerate(self.vars):
            self.c_vars[i] = _abi.pf_variable(self._names[i], v.value, v.lower, v.upper, v.step,
                                              1 if v.fixed else 0, int(v.role))
        self._keep = []
        self.c_nodes = (_abi.pf_node * max(len(self.nodes), 1))()
        for i, n in enumerate(self.nodes):
            ch = (C.c_int32 * max(len(n._desc_children), 1))(*n._desc_children)
            pa = (C.c_int32 * max(len(n._desc_params), 1))(*n._desc_params)
            ob = (C.c_int32 * max(len(n._desc_obs), 1))(*n._desc_obs)
            re = (C.c_double * max(len(n._reals), 1))(*n._reals)
            nm = n._name.encode()
            self._keep += [ch, pa, ob, re, nm]
            self.c_nodes[i] = _abi.pf_node(n.kind, nm, len(n._desc_children), ch,
                                           len(n._desc_params), pa, len(n._desc_obs), ob,
                                           len(n._reals), re, n._q)
        self.c_graph = _abi.pf_graph(len(self.vars), self.c_vars, len(self.nodes), self.c_nodes,
                                     self.root)

    def preorder(self) -> List[PdfNode]:
        """node objects in the finalized pre-order (pdf.hpp:540-549)"""
        out = []

        def walk(n):
            out.append(n)
            for c in n._children:
                walk(c)
        if self.root >= 0:
            walk(self.nodes[self.root])
        return out


def finalize(registry: ParameterRegistry, root: Optional[PdfNode], data_observables):
    """parfit::finalize (pdf.hpp:615-619): registers parameters in pre-order
    and returns the IndexTable as a list of rows [np, p..., no, col...]."""
    g = GraphDesc(root, data_observables)
    data_idx = (C.c_int32 * max(len(data_observables), 1))(*[g.var_index(o) for o in data_observables])
    return _finalize(g, registry, data_idx, len(data_observables), 0)


def _finalize(g: GraphDesc, registry, data_idx, n_data, reserved):
    st = _abi.pf_status()
    cap = 4096
    order = (C.c_int32 * cap)()
    table = (C.c_uint32 * (16 * cap))()
    n_params = C.c_int32()
    tlen = C.c_int32()
    ncols = C.c_int32()
    if lib.pf_graph_finalize(C.byref(g.c_graph), n_data, data_idx, reserved, order, cap,
                             C.byref(n_params), table, 16 * cap, C.byref(tlen), C.byref(ncols),
                             C.byref(st)):
        _raise(st)
    for i in range(n_params.value):
        registry.register_parameter(g.vars[order[i]])
    flat = list(table[: tlen.value])
    rows, k = [], 0
    while k < len(flat):
        np_ = flat[k]
        no = flat[k + 1 + np_]
        rows.append(flat[k: k + 2 + np_ + no])
        k += 2 + np_ + no
    for i, node in enumerate(g.preorder()):
        node._id = i
    return IndexTable(rows, ncols.value, n_params.value)


class IndexTable:
    """index_table.hpp:12-99 (read side)."""

    def __init__(self, rows, n_columns, n_parameters):
        self._rows = rows
        self._ncols = n_columns
        self._np = n_parameters

    def n_nodes(self):
        return len(self._rows)

    def n_columns(self):
        return self._ncols

    def n_parameters(self):
        return self._np

    def node(self, node_id):
        if node_id >= len(self._rows):
            raise Error("bad-node-id", "IndexTable::node")
        return list(self._rows[node_id])

    def param_index(self, node_id, slot):
        s = self.node(node_id)
        if slot >= s[0]:
            raise Error("out-of-bounds", "param slot")
        return s[1 + slot]

    def obs_column(self, node_id, slot):
        s = self.node(node_id)
        npar = s[0]
        if slot >= s[1 + npar]:
            raise Error("out-of-bounds", "observable slot")
        return s[2 + npar + slot]

    def __eq__(self, other):
        return (self._rows == other._rows and self._ncols == other._ncols
                and self._np == other._np)


def lookup_param(table: IndexTable, node_id, slot, params):
    gi = table.param_index(node_id, slot)
    if gi >= len(params):
        raise Error("out-of-bounds", "parameter vector shorter than index")
    return params[gi]


# ---------------------------------------------------------------------------
# engine.hpp

class MetricKind(enum.IntEnum):
    NegLogLikelihood = _abi.PF_NLL
    ChiSquared = _abi.PF_CHISQ


kPenaltyValue = 1e300
kLogFloor = 1e-300
kChiSqEps = 1e-9


class Backend:
    """engine.hpp:21-32.  Serial/Threads are accepted for source
    compatibility and select nothing: evaluation always runs on the GPU.
    ``Backend.gpus(n)`` shards events over n devices of this process."""

    def __init__(self, kind="gpu", threads=1, chunk_size=4096, devices=1, device=0, oversubscribe=False):
        self.kind = kind
        self.threads = threads
        self.chunk_size = chunk_size
        self.devices = devices
        self.device = device
        self.oversubscribe = oversubscribe

    @staticmethod
    def serial():
        return Backend("serial")

    @staticmethod
    def with_threads(n, chunk=4096):
        if n < 1:
            raise Error("bad-backend", "threads must be >= 1")
        return Backend("threads", n, chunk)

    @staticmethod
    def gpus(n=1, device=0, oversubscribe=False):
        """n devices from `device`; oversubscribe=True places shard s on
        device (device + s) mod count (the multi-device path on fewer GPUs)"""
        return Backend("gpu", devices=n, device=device, oversubscribe=oversubscribe)


class BoundModel:
    """BoundModel (engine.hpp:137-236) = GooFit's setData: the event table is
    uploaded into HBM once; eval_metric runs one CUDA graph per call."""

    def __init__(self, pdf: PdfNode, data, grid: Optional[GridSpec] = None,
                 backend: Optional[Backend] = None, shard_index: int = 0, shard_count: int = 1):
        grid = grid or GridSpec()
        backend = backend or Backend.gpus(1)
        self._pdf = pdf
        self._grid = grid
        self._binned = isinstance(data, BinnedDataSet)
        obs = data.observables()
        self._desc = GraphDesc(pdf, obs)
        table = to_event_table(data)
        self._values = np.ascontiguousarray(table, dtype=np.float64)
        self._n = self._values.shape[1] if self._values.ndim == 2 else 0
        self._total = data.total_content() if self._binned else 0.0
        self._data_idx = (C.c_int32 * max(len(obs), 1))(*[self._desc.var_index(o) for o in obs])
        cdata = _abi.pf_data(1 if self._binned else 0, len(obs), self._data_idx, self._n,
                             self._values.ctypes.data_as(C.POINTER(C.c_double)), self._total)
        opt = _abi.pf_options(backend.device, max(1, backend.devices), shard_index, shard_count, 0,
                              1 if getattr(backend, "oversubscribe", False) else 0)
        st = _abi.pf_status()
        h = C.c_void_p()
        if lib.pf_model_create(C.byref(self._desc.c_graph), C.byref(cdata), grid.points, C.byref(opt),
                               C.byref(h), C.byref(st)):
            _raise(st)
        self._h = h
        self._registry = ParameterRegistry()
        for i in range(lib.pf_model_n_params(h)):
            self._registry.register_parameter(self._desc.vars[lib.pf_model_param_variable(h, i)])
        self._nodes = self._desc.preorder()
        self._stale = False
        self._call = None
        for i, node in enumerate(self._nodes):
            node._id = i
            node._model = self
        self._table = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.pf_model_destroy(h)
            self._h = None

    def registry(self) -> ParameterRegistry:
        return self._registry

    def pdf(self):
        return self._pdf

    def grid(self):
        return self._grid

    def n_events(self) -> int:
        return int(lib.pf_model_n_events(self._h))

    def binned(self) -> bool:
        return self._binned

    def log_floor_count(self) -> int:
        return int(lib.pf_log_floor_count(self._h))

    def table(self) -> IndexTable:
        if self._table is None:
            reg = ParameterRegistry()
            self._table = _finalize(self._desc, reg, self._data_idx, len(self._data_idx),
                                    2 if self._binned else 0)
        return self._table

    def _evaluated(self):
        """norms are fetched on first use (PdfNode.cached_norm), not per call"""
        self._stale = True
        if self._nodes and self._nodes[0]._owner is not self:
            for node in self._nodes:
                node._owner = self

    def _sync_norms(self):
        self._stale = False
        n = len(self._nodes)
        norms = (C.c_double * n)()
        errs = (C.c_double * n)()
        valid = (C.c_int32 * n)()
        lib.pf_node_norms(self._h, norms, errs, valid, n)
        for i, node in enumerate(self._nodes):
            if valid[i]:
                node._norm = norms[i]
                node._norm_err = errs[i]
                node._norm_valid = True

    def eval_metric(self, params, metric=MetricKind.NegLogLikelihood, backend=None) -> float:
        p = params if (isinstance(params, np.ndarray) and params.dtype == np.float64 and params.ndim == 1
                       and params.flags.c_contiguous) else np.ascontiguousarray(params, dtype=np.float64).ravel()
        if self._call is None:  # argument objects reused by every call (the hot path of a fit)
            out, info, st = C.c_double(), _abi.pf_eval_info(), _abi.pf_status()
            self._call = (out, info, st, C.byref(out), C.byref(info), C.byref(st), _eval_fast_bound())
        out, info, st, r_out, r_info, r_st, fn = self._call
        rc = fn(self._h, p.__array_interface__["data"][0], p.size, metric, r_out, r_info, r_st)
        self._evaluated()
        if rc:
            _raise(st)
        return out.value

    def eval_metric_batch(self, params, metric=MetricKind.NegLogLikelihood) -> np.ndarray:
        p = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
        if p.ndim == 1:
            p = p.reshape(1, -1)
        out = np.empty(p.shape[0])
        st = _abi.pf_status()
        rc = lib.pf_eval_metric_batch(self._h, p.ctypes.data_as(C.POINTER(C.c_double)), p.shape[0],
                                      p.shape[1], int(metric),
                                      out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(st))
        self._evaluated()
        if rc:
            _raise(st)
        return out

    def eval_launch(self, params, metric=MetricKind.NegLogLikelihood) -> bool:
        """enqueue one evaluation on the model's stream, do not wait; True when
        the parameters are invalid (penalty, nothing enqueued).  The exact
        digits land in partial_device() for a stream-ordered collective."""
        p = np.ascontiguousarray(params, dtype=np.float64).ravel()
        pen = C.c_int32()
        st = _abi.pf_status()
        if lib.pf_eval_launch(self._h, p.ctypes.data, p.size, int(metric), C.byref(pen), C.byref(st)):
            _raise(st)
        self._evaluated()
        return bool(pen.value)

    def stream(self) -> int:
        """the model's cudaStream_t (integer), e.g. for torch.cuda.ExternalStream"""
        return int(lib.pf_model_stream(self._h))

    def partial_device(self) -> int:
        """device address of the K x 8 int64 record (6 exact digits, norm error
        word, event-error flag) the last evaluation wrote"""
        return int(lib.pf_model_partial_device(self._h))

    def group_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this model's exchange receive buffer"""
        buf = C.create_string_buffer(64)
        st = _abi.pf_status()
        if lib.pf_group_handle(self._h, buf, C.byref(st)):
            _raise(st)
        return buf.raw

    def group_join(self, world: int, rank: int, handles) -> None:
        """join a peer-memory exchange group (collective: every rank, then a
        barrier); afterwards eval_metric returns the global metric on every rank"""
        blob = b"".join(bytes(h) for h in handles)
        if len(blob) != 64 * world:
            raise Error("bad-backend", "group_join: need one 64-byte handle per rank")
        st = _abi.pf_status()
        if lib.pf_group_join(self._h, int(world), int(rank), blob, C.byref(st)):
            _raise(st)

    def eval_partial(self, params, metric=MetricKind.NegLogLikelihood):
        """(exact accumulator digits, penalty) of this process's shard"""
        p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).ravel())
        part = (C.c_int64 * _abi.PF_FX_DIGITS)()
        pen = C.c_int32()
        st = _abi.pf_status()
        if lib.pf_eval_partial(self._h, p.ctypes.data_as(C.POINTER(C.c_double)), p.size, int(metric),
                               part, C.byref(pen), C.byref(st)):
            _raise(st)
        return list(part), bool(pen.value)


# pf_eval_metric bound a second time with plain-address arguments: the
# per-call path of BoundModel.eval_metric skips ctypes pointer conversions
_eval_fast_fn = None


def _eval_fast_bound():
    global _eval_fast_fn
    if _eval_fast_fn is None:
        fn = lib["pf_eval_metric"]
        fn.restype = C.c_int
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
        _eval_fast_fn = fn
    return _eval_fast_fn


def combine_partials(parts) -> float:
    """exact combine of shard accumulators [[d0..d5], ...] (pfb200.h)"""
    flat = (C.c_int64 * (_abi.PF_FX_DIGITS * len(parts)))(*[int(v) for fx in parts for v in fx])
    return lib.pf_combine_partials(flat, len(parts))


def device_count() -> int:
    """CUDA devices visible to this process (pf_device_count)"""
    return int(lib.pf_device_count())


def kernel_launches() -> int:
    return int(lib.pf_kernel_launches())


# ---------------------------------------------------------------------------
# fit.hpp

class MinimizerKind(enum.IntEnum):
    QuasiNewton = 0
    NelderMead = 1


class FitStatus(enum.IntEnum):
    Converged = 0
    MaxIterations = 1
    Failed = 2


class FitConfig:
    """fit.hpp:23-28 (+ batch_probes: batched FD stencil on the GPU)"""

    def __init__(self, minimizer=MinimizerKind.QuasiNewton, max_iterations=10000,
                 gradient_tolerance=1e-6, simplex_tolerance=1e-8, batch_probes=True):
        self.minimizer = minimizer
        self.max_iterations = max_iterations
        self.gradient_tolerance = gradient_tolerance
        self.simplex_tolerance = simplex_tolerance
        self.batch_probes = batch_probes


class FitResult:
    """fit.hpp:32-72"""

    def __init__(self):
        self.status = FitStatus.Failed
        self.names: List[str] = []
        self.params: List[float] = []
        self.uncertainties: List[float] = []
        self.uncertainties_available = False
        self.metric_value = 0.0
        self.n_metric_calls = 0
        self.wall_time_s = 0.0
        self.grad_max_norm = math.nan

    def converged(self):
        return self.status == FitStatus.Converged

    def to_report(self) -> str:
        st = {FitStatus.Converged: "converged", FitStatus.MaxIterations: "max-iterations"}.get(
            self.status, "failed")
        lines = [f"status {st}", f"metric_value {self.metric_value:.17g}",
                 f"metric_calls {self.n_metric_calls}", f"wall_time_s {self.wall_time_s:.6g}",
                 f"grad_max_norm {self.grad_max_norm:.6g}",
                 "uncertainties " + ("available" if self.uncertainties_available else "unavailable")]
        for i, n in enumerate(self.names):
            u = self.uncertainties[i] if self.uncertainties_available else 0.0
            lines.append(f"param {n} {self.params[i]:.17g} {u:.17g}")
        return "\n".join(lines) + "\n"


def fit(bm: BoundModel, metric=MetricKind.NegLogLikelihood, backend=None,
        cfg: Optional[FitConfig] = None) -> FitResult:
    """parfit::fit (fit.hpp:498-581), run by the native driver (pf_fit)."""
    cfg = cfg or FitConfig()
    reg = bm.registry()
    ps = reg.parameters()
    n = len(ps)
    arr = lambda vals, t=C.c_double: (t * max(n, 1))(*vals)  # noqa: E731
    start = arr([p.value for p in ps])
    fixed = arr([1 if p.fixed else 0 for p in ps], C.c_int32)
    lower = arr([p.lower for p in ps])
    upper = arr([p.upper for p in ps])
    step = arr([p.step for p in ps])
    out_p = (C.c_double * max(n, 1))()
    out_u = (C.c_double * max(n, 1))()
    res = _abi.pf_fit_result(0, 0, 0.0, 0, 0.0, 0.0, out_p, out_u)
    c = _abi.pf_fit_config(int(cfg.minimizer), 1 if cfg.batch_probes else 0, cfg.max_iterations,
                           cfg.gradient_tolerance, cfg.simplex_tolerance)
    st = _abi.pf_status()
    rc = lib.pf_fit(bm._h, int(metric), C.byref(c), start, fixed, lower, upper, step, C.byref(res),
                    C.byref(st))
    bm._evaluated()  # node norms: those of the fit's last evaluation (fetched on use)
    if rc:
        _raise(st)
    r = FitResult()
    r.status = FitStatus(res.status)
    r.names = [p.name for p in ps]
    r.params = [out_p[i] for i in range(n)]
    r.uncertainties_available = bool(res.uncertainties_available)
    r.uncertainties = [out_u[i] for i in range(n)] if r.uncertainties_available else []
    r.metric_value = res.metric_value
    r.n_metric_calls = int(res.n_metric_calls)
    r.wall_time_s = res.wall_time_s
    r.grad_max_norm = res.grad_max_norm
    if r.status != FitStatus.Failed:
        reg.import_values(r.params)  # write-back (fit.hpp:556)
    return r


class FitManager:
    """GooFit-style wrapper: FitManager(pdf-bound-model).fit()"""

    def __init__(self, bm: BoundModel, metric=MetricKind.NegLogLikelihood, cfg=None):
        self.bm = bm
        self.metric = metric
        self.cfg = cfg

    def fit(self) -> FitResult:
        return fit(self.bm, self.metric, None, self.cfg)
