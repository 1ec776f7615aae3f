PFB200_DEFINES="PF_SETUP_TRACE" python - <<'PY'
import sys; sys.path.insert(0,'.')
import bench, numpy as np
from paper_1311_1753_b200 import parfit as pf
x, pdf = bench.build_model(pf)
xs = bench.make_events(1_000_000)
bm = pf.BoundModel(pdf, pf.UnbinnedDataSet.from_columns([x], xs))
p = [bench.START[v.name] for v in bm.registry().parameters()]
for i in range(3): bm.eval_metric(p)
PY
