"""Host-side logic of the engine, no GPU: graph finalization (the reference's
GraphFinalizer / IndexTable / registry contracts), datasets, the C ABI's
exported surface, NVRTC compilation of every generated evaluator for
sm_100a, and the exact superaccumulator combine."""
import ctypes as C
import os
import random
import re
import sys
from fractions import Fraction

import numpy as np
import pytest

from paper_1311_1753_b200 import _abi
from paper_1311_1753_b200 import parfit as pf

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))
from cases import CASES  # noqa: E402


# ---- variable.hpp / test_model_core.cpp -------------------------------------

def test_factories_validate():
    with pytest.raises(pf.Error, match="invalid-range"):
        pf.new_observable("x", 1, 1)
    with pytest.raises(pf.Error, match="invalid-step"):
        pf.new_parameter("p", 0, 0, 0, 1)
    with pytest.raises(pf.Error, match="invalid-range"):
        pf.new_parameter("p", 5, 0.1, 0, 1)
    x = pf.new_observable("xvar", 0, 21.49)
    assert x.role == pf.Role.Observable and x.value == 0 and x.step == 0


def test_registry_order_idempotence_collision():
    reg = pf.ParameterRegistry()
    mean = pf.new_parameter("mean", 0, 0.1, -5, 5)
    sigma = pf.new_parameter("sigma", 1, 0.1, 0.01, 5)
    assert reg.register_parameter(mean) == 0
    assert reg.register_parameter(sigma) == 1
    assert reg.register_parameter(mean) == 0
    with pytest.raises(pf.Error, match="wrong-role"):
        reg.register_parameter(pf.new_observable("x", 0, 1))
    with pytest.raises(pf.Error, match="name-collision"):
        reg.register_parameter(pf.new_parameter("mean", 1, 0.1, -5, 5))


def test_finalize_gaussian_slot_layout():
    """test_model_core.cpp:78-94: [2, 0, 1, 1, 0]"""
    x = pf.new_observable("x", -5, 5)
    g = pf.gaussian_pdf("gauss", x, pf.new_parameter("mean", 0, 0.1, -5, 5),
                        pf.new_parameter("sigma", 1, 0.1, 0.01, 5))
    table = pf.finalize(pf.ParameterRegistry(), g, [x])
    assert table.n_nodes() == 1
    assert table.node(0) == [2, 0, 1, 1, 0]


def test_finalize_product_and_shared_parameter():
    """test_model_core.cpp:102-133"""
    x, y = pf.new_observable("x", 0, 10), pf.new_observable("y", 0, 10)
    ax, ay = pf.new_parameter("alpha_x", -2.4, 0.1, -10, 10), pf.new_parameter("alpha_y", -1.1, 0.1, -10, 10)
    t = pf.finalize(pf.ParameterRegistry(), pf.prod_pdf("p", [pf.exp_pdf("ex", x, ax), pf.exp_pdf("ey", y, ay)]),
                    [x, y])
    assert t.n_nodes() == 3
    assert (t.param_index(1, 0), t.param_index(2, 0), t.obs_column(1, 0), t.obs_column(2, 0)) == (0, 1, 0, 1)
    a = pf.new_parameter("alpha", -2, 0.1, -10, 10)
    reg = pf.ParameterRegistry()
    t = pf.finalize(reg, pf.prod_pdf("p", [pf.exp_pdf("ex", x, a), pf.exp_pdf("ey", y, a)]), [x, y])
    assert reg.n_parameters() == 1 and t.param_index(1, 0) == t.param_index(2, 0)
    assert pf.lookup_param(t, 2, 0, [-3.5]) == -3.5
    with pytest.raises(pf.Error, match="out-of-bounds"):
        pf.lookup_param(t, 0, 1, [-3.5]) if t.node(0)[0] else t.param_index(0, 0)


def test_finalize_unbound_and_empty():
    x, y = pf.new_observable("x", 0, 10), pf.new_observable("y", 0, 10)
    a = pf.new_parameter("a", -2, 0.1, -10, 10)
    with pytest.raises(pf.Error, match="unbound-observable"):
        pf.finalize(pf.ParameterRegistry(), pf.exp_pdf("e", y, a), [x])
    assert pf.finalize(pf.ParameterRegistry(), None, []).n_nodes() == 0


def test_finalize_deterministic_and_mixture_order():
    """test_model_core.cpp:146-158; registry order f a m s"""
    def make():
        x = pf.new_observable("x", 0, 10)
        a, m = pf.new_parameter("a", -2, 0.1, -10, 10), pf.new_parameter("m", 5, 0.1, 0, 10)
        s, f = pf.new_parameter("s", 1, 0.1, 0.01, 5), pf.new_parameter("f", 0.5, 0.01, 0, 1)
        reg = pf.ParameterRegistry()
        t = pf.finalize(reg, pf.add_pdf("sum", [pf.exp_pdf("e", x, a), pf.gaussian_pdf("g", x, m, s)], [f]), [x])
        return t, [p.name for p in reg.parameters()]
    (t1, o1), (t2, o2) = make(), make()
    assert t1 == t2 and o1 == o2 == ["f", "a", "m", "s"]


def test_composite_synthetic_column():
    """pdf.hpp:540-560: the outer observable gets a column after the data"""
    x, u = pf.new_observable("x", 0, 10), pf.new_observable("u", 0, 10)
    a = pf.new_parameter("a", -0.5, 0.1, -10, 10)
    c0, c1 = pf.new_parameter("c0", 0, 0.1, -5, 5), pf.new_parameter("c1", 1, 0.1, -5, 5)
    t = pf.finalize(pf.ParameterRegistry(),
                    pf.composite_pdf("comp", pf.polynomial_pdf("ident", u, [c0, c1]), pf.exp_pdf("in", x, a)), [x])
    assert t.n_columns() == 2 and t.obs_column(1, 0) == 1 and t.obs_column(2, 0) == 0


def test_node_contracts():
    x = pf.new_observable("x", 0, 10)
    a = pf.new_parameter("a", -2, 0.1, -10, 10)
    f1, f2 = pf.new_parameter("f1", 0.3, 0.01, 0, 1), pf.new_parameter("f2", 0.3, 0.01, 0, 1)
    with pytest.raises(pf.Error, match="fraction-count-mismatch"):
        pf.add_pdf("s", [pf.exp_pdf("e1", x, a), pf.exp_pdf("e2", x, a)], [f1, f2])
    with pytest.raises(pf.Error, match="non-monotone"):
        pf.mapped_pdf("bad", [0, 5, 5], [pf.exp_pdf("e1", x, a), pf.exp_pdf("e2", x, a)])
    with pytest.raises(pf.Error, match="nonpositive-sigma"):
        pf.gaussian_pdf("g", x, a, pf.new_parameter("s", 1, 0.1, 0, 5))
    with pytest.raises(pf.Error, match="bad-grid"):
        pf.GridSpec(1)


# ---- dataset.hpp / test_datasets.cpp -----------------------------------------

def test_unbinned_snapshot_and_layout():
    x, y = pf.new_observable("x", 0, 10), pf.new_observable("y", 0, 10)
    ds = pf.UnbinnedDataSet([x, y])
    for xv, yv in ((1, 4), (2, 5), (3, 6)):
        x.value, y.value = xv, yv
        ds.add_event()
    x.value = 99
    assert pf.to_event_table(ds).ravel().tolist() == [1, 2, 3, 4, 5, 6]
    with pytest.raises(pf.Error, match="duplicate"):
        pf.UnbinnedDataSet([x, x])


def test_binned_edges_and_table():
    """test_datasets.cpp:66-143"""
    x = pf.new_observable("x", 0, 10)
    b = pf.BinnedDataSet([x], [10])
    b.fill([5.5])
    b.fill([1.0])
    b.fill([10.0])
    assert b.contents()[5] == 1 and b.contents()[1] == 1 and b.contents()[9] == 1
    with pytest.raises(pf.Error, match="out-of-range"):
        b.fill([10.5])
    t = pf.to_event_table(b)
    assert t.shape == (3, 10)
    assert t[0, 0] == 0.5 and t[0, 9] == 9.5 and t[2, 0] == 1.0 and t[1, 5] == 1.0


# ---- the C ABI --------------------------------------------------------------------

def test_every_declared_symbol_is_exported():
    header = open(os.path.join(ROOT, "include", "pfb200.h")).read()
    names = re.findall(r"PF_API\s+[\w\s\*]+?\b(pf_\w+)\s*\(", header)
    assert len(names) >= 20
    lib = C.CDLL(_abi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
        assert n in _abi._SIGNATURES, n
    assert lib.pf_abi_version() == 1


@pytest.mark.parametrize("name", sorted(CASES))
def test_evaluator_compiles_for_sm100a(name):
    """codegen + NVRTC (--gpu-architecture=sm_100a) for every golden case"""
    pdf, ds, grid, _ = CASES[name](pf)
    g = pf.GraphDesc(pdf, ds.observables())
    obs = (C.c_int32 * len(ds.observables()))(*[g.var_index(o) for o in ds.observables()])
    data = _abi.pf_data(1 if isinstance(ds, pf.BinnedDataSet) else 0, len(ds.observables()), obs, 0, None, 0.0)
    st, n = _abi.pf_status(), C.c_size_t()
    assert pf.lib.pf_graph_compile_check(C.byref(g.c_graph), C.byref(data), grid, C.byref(n), C.byref(st)) == 0, \
        st.message.decode()
    assert n.value > 1000


def test_argus_evaluator_compiles():
    x = pf.new_observable("x", 0, 10)
    y = pf.new_observable("y", 5.20, 5.29)
    pdf = pf.prod_pdf("c3", [pf.gaussian_pdf("g", x, pf.new_parameter("m", 5, 0.1, 0, 10),
                                             pf.new_parameter("s", 1, 0.1, 0.1, 5)),
                             pf.argus_pdf("a", y, pf.new_parameter("m0", 5.29, 0.001, 5.0, 6.0),
                                          pf.new_parameter("c", -20, 0.1, -100, 0),
                                          pf.new_parameter("p", 0.5, 0.1, 0, 5))])
    g = pf.GraphDesc(pdf, [x, y])
    obs = (C.c_int32 * 2)(g.var_index(x), g.var_index(y))
    data = _abi.pf_data(0, 2, obs, 0, None, 0.0)
    st, n = _abi.pf_status(), C.c_size_t()
    assert pf.lib.pf_graph_compile_check(C.byref(g.c_graph), C.byref(data), 1024, C.byref(n), C.byref(st)) == 0


def test_dalitz_evaluator_compiles_and_validates():
    from paper_1311_1753_b200.workloads import WORKLOADS
    W = WORKLOADS["C5TI"]
    obs, pdf = W.build(pf)
    g = pf.GraphDesc(pdf, obs)
    o = (C.c_int32 * 2)(g.var_index(obs[0]), g.var_index(obs[1]))
    data = _abi.pf_data(0, 2, o, 0, None, 0.0)
    st, n = _abi.pf_status(), C.c_size_t()
    assert pf.lib.pf_graph_compile_check(C.byref(g.c_graph), C.byref(data), 1024, C.byref(n), C.byref(st)) == 0
    m = pf.new_parameter("m", 0.77, 0.01, 0.5, 1.0)
    w = pf.new_parameter("w", 0.15, 0.01, 0.01, 0.5)
    c = pf.new_parameter("c", 1.0, 0.01, -5, 5)
    with pytest.raises(pf.Error, match="bad-channel"):
        pf.dalitz_pdf("d", obs[0], obs[1], [(m, w, c, c, 14, 1)], (1.86, 0.14, 0.14, 0.13))
    with pytest.raises(pf.Error, match="bad-kinematics"):
        pf.dalitz_pdf("d", obs[0], obs[1], [(m, w, c, c, 12, 1)], (0.3, 0.14, 0.14, 0.13))


def _digits_of(x):
    """exact superaccumulator digits of a double (python restatement of
    pf_fxl_add: value = sum d_i 2^(32 i - 128), truncation below 2^-128)"""
    fr = Fraction(x)
    sign = -1 if fr < 0 else 1
    mag = int(abs(fr) * 2 ** 128)  # truncate toward zero
    return [sign * ((mag >> (32 * i)) & 0xffffffff) for i in range(6)]


def test_exact_combine_matches_fraction_sum():
    rnd = random.Random(7)
    vals = [rnd.uniform(-1e6, 1e6) * 10 ** rnd.randint(-20, 0) for _ in range(2000)]
    shards = [vals[i::4] for i in range(4)]
    parts = []
    for sh in shards:
        acc = [0] * 6
        for v in sh:
            acc = [a + d for a, d in zip(acc, _digits_of(v))]
        parts.append(acc)
    got = pf.combine_partials(parts)
    exact = sum((Fraction(int(abs(Fraction(v)) * 2 ** 128)) * (1 if v >= 0 else -1) for v in vals),
                Fraction(0)) / 2 ** 128
    assert got == float(exact)  # correctly rounded
    # order of shards is irrelevant
    assert pf.combine_partials(parts[::-1]) == got


def test_shard_partition_covers_events():
    for n in (0, 1, 4095, 4096, 10_000_000, 100_000_003):
        for g in (1, 2, 4, 8):
            spans = []
            for r in range(g):
                first, count = C.c_uint64(), C.c_uint64()
                pf.lib.pf_shard_events(n, 1024, g, r, C.byref(first), C.byref(count))
                spans.append((first.value, count.value))
            assert spans[0][0] == 0
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1
            assert spans[-1][0] + spans[-1][1] == n
            if n > 1024 * g:
                sizes = [c for _, c in spans]
                assert max(sizes) - min(sizes) <= 1024


def test_markstein_division_is_correctly_rounded():
    """the GPU ArgusPdf log form divides by Markstein's FMA sequence on the
    per-call reciprocal: it must equal the IEEE quotient (the oracle's and the
    linear kernel's y / m0) bit for bit"""
    import ctypes as C
    import oracle
    L = oracle._olib()
    f = L.po_markstein_mismatches
    f.restype = C.c_int64
    f.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double]
    assert f(2_000_000, 1, 5.20, 5.29, 5.28, 5.30) == 0       # the C3 range
    assert f(2_000_000, 2, 1e-3, 1e3, 1e-3, 1e3) == 0         # wide operands
    assert f(1_000_000, 3, 0.5, 2.0, 1.0 - 1e-15, 1.0 + 1e-15) == 0  # near-1 divisors


def test_event_store_text_and_binary(tmp_path):
    """dataset.hpp:184-245 text format (same header checks and error codes) and
    the binary SoA store; both round-trip the event table bit for bit"""
    x = pf.new_observable("x", 0, 10)
    y = pf.new_observable("y", -1, 1)
    rng = np.random.default_rng(4)
    cols = np.stack([10 * rng.random(1000), rng.uniform(-1, 1, 1000)])
    cols[0, :3] = [0.1, 1.0 / 3.0, 5e-324]
    ds = pf.UnbinnedDataSet.from_columns([x, y], cols)
    pf.write_text_file(ds, str(tmp_path / "ev.txt"))
    back = pf.read_text_file(str(tmp_path / "ev.txt"), [x, y])
    assert np.array_equal(back.columns(), cols)
    pf.write_binary_file(ds, str(tmp_path / "ev.bin"))
    assert np.array_equal(pf.read_binary_file(str(tmp_path / "ev.bin"), [x, y]).columns(), cols)
    with pytest.raises(pf.Error, match="bad-format"):
        pf.read_text_file(str(tmp_path / "ev.txt"), [y, x])  # header order
    (tmp_path / "short.txt").write_text("# x y\n1 2\n3\n")
    with pytest.raises(pf.Error, match="bad-format: short row"):
        pf.read_text_file(str(tmp_path / "short.txt"), [x, y])
    with pytest.raises(pf.Error, match="io-error"):
        pf.read_text_file(str(tmp_path / "missing.txt"), [x, y])


def test_event_store_text_matches_reference_writer(tmp_path):
    """our writer's bytes equal the reference's write_text (dataset.hpp:187-200),
    compiled from the reference headers (skipped where they are absent)"""
    import shutil
    import subprocess
    inc = "/root/reference/proj/include"
    if not os.path.isdir(inc) or not shutil.which("g++"):
        pytest.skip("reference headers not present")
    src = tmp_path / "w.cpp"
    src.write_text(
        '#include <iostream>\n#include "parfit/dataset.hpp"\n#include "parfit/variable.hpp"\n'
        "using namespace parfit;\nint main() {\n"
        '  auto x = new_observable("x", 0, 10); auto y = new_observable("y", -1, 1);\n'
        "  UnbinnedDataSet ds({x, y});\n"
        "  double vals[4][2] = {{0.1, -0.5}, {1.0 / 3.0, 0.25}, {5e-324, 1e300}, {9.999999999999998, -1}};\n"
        "  for (auto& v : vals) { x->value = v[0]; y->value = v[1]; ds.add_event(); }\n"
        "  write_text(ds, std::cout);\n}\n")
    exe = tmp_path / "w"
    r = subprocess.run(["g++", "-std=gnu++20", "-I", inc, str(src), "-o", str(exe)], capture_output=True, text=True)
    if r.returncode:
        pytest.skip("reference headers do not build here: " + r.stderr[:200])
    ref = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    x = pf.new_observable("x", 0, 10)
    y = pf.new_observable("y", -1, 1)
    ds = pf.UnbinnedDataSet.from_columns([x, y], np.array([[0.1, 1.0 / 3.0, 5e-324, 9.999999999999998],
                                                         [-0.5, 0.25, 1e300, -1.0]]))
    import io
    buf = io.StringIO()
    pf.write_text(ds, buf)
    assert buf.getvalue() == ref


def test_toy_rng_is_the_reference_stream():
    """ToyRng (generate.hpp:19-27) == the oracle's mt19937_64 recipe"""
    import oracle
    r = pf.ToyRng(7)
    got = np.array([r.uniform() for _ in range(2000)])
    assert np.array_equal(got, oracle.mt64_uniform(7, 2000))
    r = pf.ToyRng(7)
    assert all(-3.0 <= r.uniform(-3, 5) < 5.0 for _ in range(500))


def test_generate_events_rejects_empty_request_without_a_gpu():
    """test_generate.cpp:141-146: checked before any device work"""
    x = pf.new_observable("x", 0, 10)
    pdf = pf.exp_pdf("e", x, pf.new_parameter("a", -0.5, 0.1, -5, 5))
    with pytest.raises(pf.Error, match="bad-arity: generate_events: n_events"):
        pf.generate_events(pdf, [x], 0, 1)


def test_mt_jump_table_jumps_the_reference_stream():
    """csrc/mt_jump_table.inc (tools/gen_mt_jump.py): applying g_k (Horner in
    blocks of 156 coefficients, the GPU generator's algorithm) to a window of
    the mt19937_64 stream lands exactly k J words further on."""
    import importlib.util
    import re as _re
    spec = importlib.util.spec_from_file_location("gen_mt_jump", os.path.join(ROOT, "tools", "gen_mt_jump.py"))
    gj = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gj)
    text = open(os.path.join(ROOT, "paper_1311_1753_b200", "csrc", "mt_jump_table.inc")).read()
    rows = _re.findall(r"\{([0-9a-fx,ul]+)\}", text)
    assert len(rows) == gj.SEGMENTS + 1
    k = 3
    words = [int(w.rstrip("ul"), 16) for w in rows[k].split(",")]
    g = sum(w << (64 * i) for i, w in enumerate(words))
    base = gj.stream(gj.seed_state(20260823), gj.N)  # a window in the image of T
    far = base + gj.stream(base, k * gj.JUMP + gj.N)
    assert gj.apply_poly(g, base) == far[k * gj.JUMP: k * gj.JUMP + gj.N]
