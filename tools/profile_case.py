"""ncu driver: run a golden case (tests/cases.py) through the GPU path."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import cases
import paper_2308_16395_b200.streaming as S
case = cases.STREAM_CASES[sys.argv[1] if len(sys.argv) > 1 else "c3_40"]()
st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
for s in case.slices[:8]:
    st.stream_update(s)
st.synchronize()
print("ok", st.query()["core_dims"])
