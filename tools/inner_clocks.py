"""Phase clocks of isvd_inner_kernel's wide path (33..64 columns) late in C5."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
L = S.load_library()
cfg = dg.CONFIGS["c5"]
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
st = S.StreamingState(device=0, asynchronous=False)
st.init_flat(torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)]), gen.init_dims(), cfg.tau)
for i in range(350):
    st.stream_update(gen.slice_torch(cfg.n_init + i, dev))
st.synchronize()
c = np.zeros(32, dtype=np.int64)
L.tsg_debug_isvd_clocks(c.ctypes.data_as(ctypes.c_void_p))
f = lambda a, b: f"{(c[a] - c[b]) / 1965:7.1f} us"
print("ranks", st.query()["core_dims"])
print("partial sums", f(1, 0), "| pre", f(4, 1), "| secular (wide)", f(5, 4), "| truncate", f(6, 5),
      "| U fill", f(17, 6), "| MGS", f(7, 17), "| M, w, stores", f(2, 7), "| total", f(2, 0))
print("wide secular: prologue + deflation", f(10, 4), "| roots", f(11, 10), "| z-hat, all eigenvalues, sort", f(12, 11),
      "| vectors", f(5, 12))
