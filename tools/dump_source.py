"""Generated evaluator source for a workload (no GPU needed):
  python tools/dump_source.py C2 > /tmp/c2.cu"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1753_b200 import parfit as pf, _abi  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402

W = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
obs, pdf = W.build(pf)
g = pf.GraphDesc(pdf, obs)
o = (C.c_int32 * len(obs))(*[g.var_index(x) for x in obs])
binned = 1 if (getattr(W, "binned", False) or W.metric == 1) else 0
data = _abi.pf_data(binned, len(obs), o, 0, None, 0.0)
st, n = _abi.pf_status(), C.c_size_t()
buf = C.create_string_buffer(1 << 22)
rc = pf.lib.pf_graph_codegen(C.byref(g.c_graph), C.byref(data), W.grid, buf, 1 << 22, C.byref(n), C.byref(st))
assert rc == 0, st.message.decode()
sys.stdout.write(buf.value.decode())
