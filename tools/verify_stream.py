"""Stream a config on the device, then verify every slice's reconstruction
error against the regenerated slice (device reconstruct), next to the ledger
estimate. usage: python tools/verify_stream.py c4 [n_stream] [size]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
name = sys.argv[1]
nst = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = dg.CONFIGS[name]
if len(sys.argv) > 3:
    sz = int(sys.argv[3])
    cfg = dg.scaled(cfg, (sz,) * (len(cfg.slice_dims) - 1) + cfg.slice_dims[-1:] if name == "c4" else (sz,) * len(cfg.slice_dims))
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
init = torch.empty(cfg.n_init * cfg.slice_elems, dtype=torch.float64, device=dev)
for t in range(cfg.n_init):
    init[t * cfg.slice_elems:(t + 1) * cfg.slice_elems] = gen.slice_torch(t, dev)
st = S.StreamingState(device=0, asynchronous=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
del init
print("after init", st.query()["core_dims"], "est", st.estimate_relative_error())
for t in range(cfg.n_init, cfg.n_init + nst):
    st.stream_update(gen.slice_torch(t, dev))
    st.synchronize()
    m = st.last_metrics()
    print("t", t, m["ranks"], "mask", m["expanded_mask"], "est", "%.3e" % m["error_estimate"],
          "|y| %.4e" % m["slice_norm"], "res", " ".join("%.4e" % v for v in m["mode_residuals"]),
          "proj %.6e" % m["projected_norm"])
    if os.environ.get("ORTH"):
        e = st.export()
        print("   orth defects", ["%.1e" % np.max(np.abs(f.T @ f - np.eye(f.shape[1]))) for f in e.factors],
              "right %.1e" % np.max(np.abs(e.right.T @ e.right - np.eye(e.rank))))
q = st.query()
errs = []
for t in range(q["n_d"]):
    y = gen.slice_torch(t, dev)
    a, b = st.error_sums(y, t, 1)
    errs.append((a / b) ** 0.5)
print("per-slice relative error:", " ".join("%.2e" % e for e in errs))
print("estimate %.3e" % st.estimate_relative_error())
