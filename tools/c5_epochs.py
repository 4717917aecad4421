"""C5 (rank-growth stress, 256^3) whole stream on the device: wall time per
block of 25 updates, ranks, and the slow-path count.  Usage: c5_epochs.py [n_updates]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2308_16395_b200.streaming as S
from paper_2308_16395_b200 import datagen as dg
cfg = dg.CONFIGS["c5"]
nup = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n_slices - cfg.n_init
gen = dg.make_stream(cfg)
dev = torch.device("cuda", 0)
init = torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)])
st = S.StreamingState(device=0, asynchronous=True)
st.init_flat(init, gen.init_dims(), cfg.tau)
del init
blk = 25
tot = 0.0
for b0 in range(0, nup, blk):
    ys = [gen.slice_torch(cfg.n_init + b0 + i, dev) for i in range(min(blk, nup - b0))]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for y in ys:
        st.stream_update(y)
    st.synchronize()
    dt = time.perf_counter() - t0
    tot += dt
    q = st.query()
    ms = st.metrics()[-len(ys):]
    grown = sum(1 for m in ms if m["expanded_mask"])
    print(f"slices {cfg.n_init + b0:3d}..{cfg.n_init + b0 + len(ys) - 1:3d}: {dt * 1e3 / len(ys):8.3f} ms/slice, "
          f"ranks {q['core_dims']}, n = {int(np.prod(q['core_dims'][:-1]))}, grown on {grown} slices", flush=True)
print(f"whole stream: {nup} updates in {tot * 1e3:.1f} ms = {nup / tot:.0f} slices/s, "
      f"estimate {st.estimate_relative_error():.3e}")
