"""Average in-kernel phase clocks of the cluster insertion kernel over a whole
pipelined C2 stream (contended: mode 0 and tails of the following slices run
beside it), against the last insertion (uncontended)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
L = S.load_library()
cfg = dg.CONFIGS["c2"]
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
st = S.StreamingState(device=0, asynchronous=os.environ.get("TL_SYNC") is None)
st.init_flat(torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)]), gen.init_dims(), cfg.tau)
ys = [gen.slice_torch(cfg.n_init + i, dev) for i in range(80)]
for y in ys[:20]:
    st.stream_update(y)
st.synchronize()
a0 = np.zeros(32, dtype=np.int64); a0[0] = -12345
L.tsg_debug_isvd_clocks(a0.ctypes.data_as(ctypes.c_void_p))
for y in ys[20:]:
    st.stream_update(y)
st.synchronize()
a1 = np.zeros(32, dtype=np.int64); a1[0] = -12345
L.tsg_debug_isvd_clocks(a1.ctypes.data_as(ctypes.c_void_p))
d = a1 - a0
n = max(int(d[31]), 1)
c = d / n
names = [(8, "entry/Q loads"), (1, "CGS2 passes"), (4, "pre-inner"), (5, "secular"), (6, "truncate"), (7, "U+MGS"),
         (2, "barrier"), (16, "M+sw"), (14, "row updates"), (15, "left"), (3, "cluster reduce"), (9, "publish")]
prev = 0.0
print(f"cluster insertion kernel, average over {n} insertions (cycles at 1.965 GHz -> us)")
for i, nm in names:
    print(f"  {nm:16s} {c[i] - prev:9.0f} cycles  {(c[i] - prev) / 1965:6.2f} us")
    prev = c[i]
print(f"  total body       {c[9]:9.0f} cycles  {c[9] / 1965:6.2f} us")
