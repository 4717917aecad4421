"""Bitwise reproducibility of the growth case across modes/runs (debug aid)."""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import cases
from paper_2308_16395_b200 import streaming as S

def run(asyn):
    case = cases.case_growth()
    st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims, asynchronous=asyn)
    out = []
    for s in case.slices:
        st.stream_update(s)
        if not asyn:
            out.append(st.export().core.copy())
    st.synchronize()
    return st.export(), out, [m["ranks"] for m in st.metrics()], [m["expanded_mask"] for m in st.metrics()]

a1, _, ra, ma = run(True)
a2, _, _, _ = run(True)
s1, traj, rs, ms = run(False)
s2, _, _, _ = run(False)
print("async==async", np.array_equal(a1.core, a2.core), "sync==sync", np.array_equal(s1.core, s2.core),
      "async==sync", np.array_equal(a1.core, s1.core))
print("ranks equal", ra == rs, "masks", ma)
print("max diff", np.max(np.abs(a1.core - s1.core)) if a1.core.shape == s1.core.shape else "shape")

def metr(asyn):
    case = cases.case_growth()
    st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims, asynchronous=asyn)
    for s in case.slices:
        st.stream_update(s)
    st.synchronize()
    return st.metrics()

m1, m2, m3 = metr(True), metr(True), metr(False)
for name, other in (("async2", m2), ("sync", m3)):
    first = None
    for i, (x, y) in enumerate(zip(m1, other)):
        for key in ("slice_norm", "projected_norm", "error_estimate", "trunc_margin", "mode_residuals"):
            if np.any(np.asarray(x[key]) != np.asarray(y[key])):
                first = (i, key, x[key], y[key])
                break
        if first:
            break
    print("first diff vs", name, first)
