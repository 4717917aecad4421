"""Per-step / per-mode residual comparison GPU vs oracle on reduced C4."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import cases, py_oracle
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
size = int(sys.argv[1]) if len(sys.argv) > 1 else 48
cfg = dg.scaled(dg.CONFIGS["c4"], (size, size, size, 16), n_slices=16, n_init=10)
case = cases.config_case(cfg)
st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
orc = py_oracle.load_oracle()
ho = orc.stream_init(case.init_flat.reshape(case.init_dims[::-1]).transpose(), case.tau)
for y in case.slices:
    st.stream_update(y)
    ho.update_flat(y)
mg, mo = st.metrics(), ho.metrics()
for a, b in zip(mg[-len(case.slices):], mo[-len(case.slices):]):
    ra, rb = np.array(a["mode_residuals"]), np.array(b["mode_residuals"])
    print(a["slice_index"], a["expanded_mask"], b["expanded_mask"], a["ranks"],
          " ".join(f"{x:.6e}/{(x-y)/max(y,1e-300):+.1e}" for x, y in zip(ra, rb)),
          f"|y|={a['slice_norm']:.4e}")
