"""Sync-mode result with and without an inflated r_hint (debug aid)."""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
if len(sys.argv) > 1:
    import cases
    from paper_2308_16395_b200 import streaming as S
    case = cases.case_growth() if sys.argv[2] == "growth" else cases.STREAM_CASES[sys.argv[2]]()
    st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
    k = int(sys.argv[3]) if len(sys.argv) > 3 else len(case.slices)
    for s in case.slices[:k]:
        st.stream_update(s)
    e = st.export()
    np.savez(sys.argv[1], core=e.core, left=e.left, right=e.right, sigma=e.sigma)
    sys.exit(0)
for case in ("growth", "c1"):
    for k in (11, 12, 20, 1000):
        subprocess.run([sys.executable, __file__, "/tmp/a.npz", case, str(k)], check=True)
        subprocess.run([sys.executable, __file__, "/tmp/b.npz", case, str(k)], check=True, env=dict(os.environ, TSG_RHINT_PAD="4"))
        a, b = np.load("/tmp/a.npz"), np.load("/tmp/b.npz")
        print(case, k, {key: (np.array_equal(a[key], b[key]), float(np.max(np.abs(a[key] - b[key]))) if a[key].shape == b[key].shape else "shape") for key in ("core", "left", "right", "sigma")})
