import sys, os, time, traceback
sys.path.insert(0, "."); sys.path.insert(0, "oracle"); sys.path.insert(0, "tests")
import numpy as np
import cases, parity as P
from conftest import load_golden
import paper_2308_16395_b200.streaming as S
for name in sorted(cases.STREAM_CASES):
    try:
        case = cases.STREAM_CASES[name]()
        g = load_golden("stream_" + name)
        t0 = time.time()
        st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
        for s in case.slices: st.stream_update(s)
        st.synchronize()
        t1 = time.time()
        sg = st.export()
        mc = P.compare_metrics(P.metrics_arrays(st.metrics(), sg.order), P.golden_metrics(g), float(g["total_input_sq"]))
        sc = P.compare_states(sg, P.state_from_golden(g))
        print(name, f"{t1-t0:.2f}s", sg.core_dims, tuple(g["core_dims"]), mc, sc, flush=True)
    except Exception as e:
        traceback.print_exc()
