"""GPU vs oracle on a config-4 stream with a chosen slice shape."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import cases, py_oracle, parity as P
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
dims = tuple(int(v) for v in sys.argv[1].split(","))
nst = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = dg.scaled(dg.CONFIGS["c4"], dims, n_slices=10 + nst, n_init=10)
case = cases.config_case(cfg)
st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
ho = py_oracle.load_oracle().stream_init(case.init_flat.reshape(case.init_dims[::-1]).transpose(), case.tau)
prevR = None
for y in case.slices:
    prev = st.export().factors[0] if os.environ.get("PRE") else None
    st.stream_update(y)
    ho.update_flat(y)
    a, b = st.last_metrics(), ho.metrics()[-1]
    e = st.export()
    print(a["ranks"], b["ranks"], "res", ["%.4e/%.4e" % (x, z) for x, z in zip(a["mode_residuals"], b["mode_residuals"])],
          "orth", ["%.1e" % np.max(np.abs(f.T @ f - np.eye(f.shape[1]))) for f in e.factors])
    u = e.factors[0]; r0 = prev.shape[1] if prev is not None else u.shape[1]
    if u.shape[1] > r0:
        w = u[:, r0:]
        print("   old cols unchanged:", np.array_equal(u[:, :r0], prev),
              "old-old %.1e" % np.max(np.abs(prev.T @ prev - np.eye(r0))),
              "new-new %.1e" % np.max(np.abs(w.T @ w - np.eye(w.shape[1]))),
              "old-new %.1e" % np.max(np.abs(prev.T @ w)), "new norms", np.round(np.linalg.norm(w, axis=0), 4)[:6])
