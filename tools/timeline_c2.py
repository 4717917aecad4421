"""Per-slice event timeline of the async engine on C2 (TSG_PROFILE):
mode-0 start/end, decision (tail end), insertion start/end, in us."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
cfg = dg.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
init = torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)])
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # untimed updates before the window
st = S.StreamingState(device=0, asynchronous=os.environ.get("TL_SYNC") is None, profile=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
del init
for i in range(skip):
    st.stream_update(gen.slice_torch(cfg.n_init + i, dev))
    if i % 8 == 7:
        st.synchronize()
st.synchronize()
ys = [gen.slice_torch(cfg.n_init + skip + i, dev) for i in range(50)]
for y in ys[:20]:
    st.stream_update(y)
st.synchronize()
st.profile(reset=True)
import time
t0 = time.perf_counter()
for y in ys[20:]:
    st.stream_update(y)
st.synchronize()
print("host wall per update: %.1f us; ranks %s" % ((time.perf_counter() - t0) / 30 * 1e6, st.query()["core_dims"]))
t = st.timeline() * 1e3
t -= t[0, 0]
print("slice  m0_start  m0_end  decision  isvd_start  isvd_end | m0  tail  dec->isvd  isvd  isvd_gap")
prev_end = None
for i, r in enumerate(t):
    gap = r[3] - prev_end if prev_end is not None else float("nan")
    print("%3d %9.1f %8.1f %9.1f %10.1f %9.1f | %5.1f %5.1f %8.1f %6.1f %6.1f" %
          (i, r[0], r[1], r[2], r[3], r[4], r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], gap))
    prev_end = r[4]
d = np.diff(t[:, 4])
print("period (isvd end to end) mean %.1f us" % d.mean())
