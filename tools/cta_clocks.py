"""Phase clocks of the single-CTA insertion (isvd_cta_kernel) after a C2 run
through the async engine (cycles, thread 0 of the CTA)."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
L = S.load_library()
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = dg.CONFIGS[name]
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
init = torch.empty(cfg.n_init * cfg.slice_elems, dtype=torch.float64, device=dev)
for t in range(cfg.n_init):
    init[t * cfg.slice_elems:(t + 1) * cfg.slice_elems] = gen.slice_torch(t, dev)
st = S.StreamingState(device=0, asynchronous=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
ys = [gen.slice_torch(cfg.n_init + i, dev) for i in range(24)]
torch.cuda.synchronize()
for y in ys:
    st.stream_update(y)
st.synchronize()
c = np.zeros(32, dtype=np.int64)
L.tsg_debug_isvd_clocks(c.ctypes.data_as(ctypes.c_void_p))
d = lambda a, b: int(c[b] - c[a])
print(name, st.query()["core_dims"], "fallbacks", int(c[26]))
print("entry", d(0, 8), "cgs2", d(8, 1), "pre", d(1, 4), "inner", d(4, 7), "sync", d(7, 2),
      "M", d(2, 16), "rows", d(16, 14), "left", d(14, 15), "reduce", d(15, 3), "record", d(3, 9), "total", d(0, 9))
print("inner: deflate-check", d(4, 10), "roots", d(10, 11), "zhat", d(11, 12), "vectors", d(12, 13),
      "trunc", d(13, 5), "U", d(5, 6), "cgs+out", d(6, 7))
