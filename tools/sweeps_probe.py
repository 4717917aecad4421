import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import cases
from paper_2308_16395_b200 import datagen as dg, streaming as S
cfg = dg.CONFIGS["c2"]
case = cases.config_case(cfg, n_slices=cfg.n_init + 20)
st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
for s in case.slices: st.stream_update(s)
print([m["jacobi_sweeps"] for m in st.metrics()])
print([m["ranks"][-1] for m in st.metrics()])
