"""Lean driver for ncu: init a config on cuda:0 and run a few updates."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_16395_b200 import datagen as dg  # noqa: E402
from paper_2308_16395_b200 import streaming as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--updates", type=int, default=6)
ap.add_argument("--async-mode", action="store_true")
args = ap.parse_args()
cfg = dg.CONFIGS[args.config]
gen = dg.TuckerStream(cfg)
dev = torch.device("cuda", 0)
init = torch.cat([gen.slice_torch(t, dev) for t in range(cfg.n_init)])
slices = [gen.slice_torch(cfg.n_init + i, dev) for i in range(args.updates)]
torch.cuda.synchronize()
st = S.StreamingState(device=0, asynchronous=args.async_mode)
st.init_flat(init, gen.init_dims(), cfg.tau)
for s in slices:
    st.stream_update(s)
st.synchronize()
print("ranks", st.query()["core_dims"], "launches", st.kernel_launches())
