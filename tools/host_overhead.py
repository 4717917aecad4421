"""Host-side cost per stream_update vs device time (C2, async engine)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2308_16395_b200 import datagen as dg, streaming as S
cfg = dg.CONFIGS["c2"]; gen = dg.TuckerStream(cfg); dev = torch.device("cuda", 0)
init = torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)])
slices = [gen.slice_torch(cfg.n_init + i, dev) for i in range(60)]
torch.cuda.synchronize()
st = S.StreamingState(device=0, asynchronous=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
for i in range(5): st.stream_update(slices[i])
st.synchronize()
ptr = [s.data_ptr() for s in slices]
t0 = time.perf_counter()
for i in range(5, 55): st.update_device_ptr(ptr[i])
t1 = time.perf_counter()
st.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6*(t1-t0)/50:.1f} us/update, total {1e6*(t2-t0)/50:.1f} us/update")
# raw ctypes call (no Python wrapper logic)
import ctypes as C
L = st.L
h = st.h
fn = L.tsg_update
t0 = time.perf_counter()
for i in range(5, 55): fn(h, C.c_void_p(ptr[i]), 1)
t1 = time.perf_counter()
st.synchronize()
print(f"raw ctypes enqueue {1e6*(t1-t0)/50:.1f} us/update")
# cost of one trivial CUDA API call from here
t0 = time.perf_counter()
for i in range(200): torch.cuda.current_stream().query()
t1 = time.perf_counter()
print(f"stream query {1e6*(t1-t0)/200:.2f} us")
