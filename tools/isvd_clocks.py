"""Print the fused-ISVD phase clocks (g_isvd_clk) after a few updates of a case."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import cases
import paper_2308_16395_b200.streaming as S
L = S.load_library()
name = sys.argv[1] if len(sys.argv) > 1 else "c3_40"
if name in ("c2", "c3", "c5"):
    from paper_2308_16395_b200 import datagen as dg
    cfg = dg.CONFIGS[name]
    case = cases.config_case(cfg, n_slices=cfg.n_init + 8)
else:
    case = cases.STREAM_CASES[name]()
asyn = bool(os.environ.get("ASYNC"))
if asyn and name in ("c2", "c3", "c5"):
    # device-resident slices through the async engine (the insertion overlaps
    # the next slices' projections): clocks of the last insertion
    import torch
    dev = torch.device("cuda", 0)
    gen = dg.make_stream(cfg)
    st = S.StreamingState(device=0, asynchronous=True)
    st.init_flat(torch.as_tensor(case.init_flat, device=dev), case.init_dims, case.tau)
    ys = [gen.slice_torch(cfg.n_init + i, dev) for i in range(30)]
    for y in ys:
        st.stream_update(y)
    st.synchronize()
else:
    st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
    for s in case.slices[:8]:
        st.stream_update(s)
c = np.zeros(32, dtype=np.int64)
L.tsg_debug_isvd_clocks(c.ctypes.data_as(ctypes.c_void_p))
print(name, st.query()["core_dims"], "pgram", c[8] - c[0], "passes", c[1] - c[8], "pre", c[4] - c[1],
      "secular", c[5] - c[4], "trunc", c[6] - c[5], "U+MGS", c[7] - c[6], "tail", c[2] - c[7],
      "update", c[3] - c[2], "finalize", c[9] - c[3], "total", c[9] - c[0])
print("small-kernel view: entry/Q", c[8] - c[0], "cgs2", c[1] - c[8], "pre-inner", c[4] - c[1],
      "inner(warp0)", c[7] - c[4], "barrier", c[2] - c[7], "update+left", c[3] - c[2], "publish", c[9] - c[3],
      "total", c[9] - c[0])
print("secular: prologue", c[10] - c[4], "roots", c[11] - c[10], "zhat+lam", c[12] - c[11], "sort", c[13] - c[12],
      "vectors", c[5] - c[13], "| trunc", c[6] - c[5], "U+MGS", c[7] - c[6])
print("update rows", c[14] - c[2], "left", c[15] - c[14], "reduce", c[3] - c[15])
print("M+sw", c[16] - c[2], "wait+sync", c[17] - c[16], "row0", c[18] - c[17], "row1", c[14] - c[18])
print("grid leader: M+inv", c[16] - c[2], "handoff", c[17] - c[16], "own rows", c[18] - c[17], "left", c[14] - c[18], "reduce+publish", c[9] - c[14])
print("own rows: e", c[19] - c[17], "chunk0", c[20] - c[19], "chunk1", c[18] - c[20])
print("prologue: ctrl/slot/commit %d, barrier %d, prefetch issue %d" % (c[21] - c[0], c[22] - c[21], c[8] - c[22]))
print("grid kernel wall (leader entry -> last CTA publish): %.2f us" % ((c[25] - c[24]) * 1e-3))
