"""Phase timing (TSG_PROFILE) of the C2 engine in synchronous vs async mode:
does the insertion take longer when it overlaps the next slices' projections?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
cfg = dg.CONFIGS["c2"]
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
init = torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)])
ys = [gen.slice_torch(cfg.n_init + i, dev) for i in range(60)]
for asyn in (False, True):
    st = S.StreamingState(device=0, asynchronous=asyn, profile=True)
    st.init_flat(init, gen.init_dims(), cfg.tau)
    for y in ys[:20]:
        st.stream_update(y)
    st.synchronize()
    st.profile(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for y in ys[20:]:
        st.stream_update(y)
    st.synchronize()
    e1.record()
    torch.cuda.synchronize()
    p = st.profile()
    print("async" if asyn else "sync ", "%.1f us/slice" % (e0.elapsed_time(e1) * 1e3 / 40),
          {k: round(v * 1e3, 1) for k, v in p.items() if k != "updates"})
    st.close()
