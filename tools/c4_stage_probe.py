"""Full-size C4 first update with per-stage host RSS / device memory prints
(diagnoses where the parity test's host memory goes)."""
import os, sys, time, resource
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
import py_oracle
T0 = time.time()
def stage(msg):
    rss = int(open(f"/proc/{os.getpid()}/statm").read().split()[1]) * 4096 / 1e9
    free, tot = torch.cuda.mem_get_info()
    print(f"[{time.time()-T0:7.1f}s] {msg}: rss {rss:.1f} GB, gpu used {(tot-free)/1e9:.1f} GB, torch alloc {torch.cuda.memory_allocated()/1e9:.1f}", flush=True)
dev = torch.device("cuda", 0)
cfg = dg.CONFIGS["c4"]
gen = dg.make_stream(cfg)
stage("start")
init = torch.empty(cfg.n_init * cfg.slice_elems, dtype=torch.float64, device=dev)
for t in range(cfg.n_init):
    init[t * cfg.slice_elems:(t + 1) * cfg.slice_elems] = gen.slice_torch(t, dev)
    stage(f"init slice {t}")
st = S.StreamingState(device=0, asynchronous=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
stage("gpu init done")
del init
torch.cuda.empty_cache()
e = st.export()
stage(f"export ranks {e.core_dims}")
chk = py_oracle.load_reference() if py_oracle.reference_available() else py_oracle.load_oracle()
ho = chk.assemble(py_oracle.State(order=e.order, n_d=e.n_d, rank=e.rank, insertions=e.insertions,
                           core_dims=e.core_dims, slice_dims=e.slice_dims, tau=e.tau,
                           squared_error=e.squared_error, total_input_sq=e.total_input_sq,
                           nonstream_discarded_sq=e.nonstream_discarded_sq, core=e.core,
                           factors=e.factors, sigma=e.sigma, left=e.left, right=e.right))
stage("assembled")
y = gen.slice_torch(cfg.n_init, dev)
st.stream_update(y); st.synchronize()
stage("gpu update done")
yh = y.cpu().numpy()
stage("slice on host")
import threading
stop = False
def mon():
    while not stop:
        time.sleep(2); stage("  ... reference update running")
th = threading.Thread(target=mon, daemon=True); th.start()
ho.update_flat(yh)
stop = True
stage("reference update done")
