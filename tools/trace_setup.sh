#!/bin/bash
# Per-phase clock64 stamps of the setup kernel (PF_SETUP_TRACE) for a
# workload (default C2), printed by block 0 on three evaluations.
CFG=${1:-C2}
PFB200_DEFINES="PF_SETUP_TRACE" python - "$CFG" <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1311_1753_b200 import parfit as pf
from paper_1311_1753_b200.workloads import WORKLOADS
W = WORKLOADS[sys.argv[1]]
obs, pdf = W.build(pf)
bm = pf.BoundModel(pdf, W.data(pf, obs, 100_000))
p = W.params(bm)
for i in range(3):
    bm.eval_metric(p)
PY
