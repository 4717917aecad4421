import sys; sys.path.insert(0,"."); sys.path.insert(0,"tests")
import cases, paper_2308_16395_b200.streaming as S
for name in ["thin", "growth24", "order2"]:
    case = cases.STREAM_CASES[name]()
    try:
        st = S.stream_init(case.init_flat, case.tau, dims=case.init_dims)
        for i, s in enumerate(case.slices):
            st.stream_update(s)
        print(name, "ok", st.query()["core_dims"])
    except Exception as e:
        print(name, "slice", i, "FAILED", e)
