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
st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
for s in case.slices[:8]:
    st.stream_update(s)
c = np.zeros(16, dtype=np.int64)
L.tsg_debug_isvd_clocks(c.ctypes.data_as(ctypes.c_void_p))
print(name, st.query()["core_dims"], "pgram", c[8] - c[0], "passes", c[1] - c[8], "pre", c[4] - c[1],
      "secular", c[5] - c[4], "trunc", c[6] - c[5], "U+MGS", c[7] - c[6], "tail", c[2] - c[7],
      "update", c[3] - c[2], "finalize", c[9] - c[3], "total", c[9] - c[0])
