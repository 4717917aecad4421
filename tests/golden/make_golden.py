"""Generate the golden fixtures from the REFERENCE itself.

Runs oracle/_ref/libtucker_ref.so — the reference's own sources compiled in
place from /root/reference by oracle/Makefile — on the deterministic cases of
tests/cases.py and stores its outputs (final streaming state, per-slice
metrics, building-block results) plus a checksum of the inputs. Run here
(the reference exists only in this container):

    make -C oracle all ref && python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import cases  # noqa: E402
import py_oracle as po  # noqa: E402


def input_digest(case) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(case.init_flat).tobytes())
    for s in case.slices:
        h.update(np.ascontiguousarray(s).tobytes())
    return h.hexdigest()


def stream_fixture(ref, case) -> dict:
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    h = ref.stream_init(x, case.tau)
    for s in case.slices:
        h.update_flat(s)
    st = h.export()
    ms = h.metrics()
    d = st.order
    out = {
        "digest": np.array(input_digest(case)),
        "order": st.order, "n_d": st.n_d, "rank": st.rank, "insertions": st.insertions,
        "core_dims": np.array(st.core_dims), "slice_dims": np.array(st.slice_dims),
        "tau": st.tau, "squared_error": st.squared_error, "total_input_sq": st.total_input_sq,
        "nonstream_discarded_sq": st.nonstream_discarded_sq,
        "core": st.core, "sigma": st.sigma, "left": st.left, "right": st.right,
        "estimate": h.estimate_relative_error(),
        "m_ranks": np.array([m["ranks"] for m in ms]).reshape(len(ms), d),
        "m_slice_norm": np.array([m["slice_norm"] for m in ms]),
        "m_projected_norm": np.array([m["projected_norm"] for m in ms]),
        "m_error_estimate": np.array([m["error_estimate"] for m in ms]),
        "m_mode_residuals": np.array([m["mode_residuals"] for m in ms]).reshape(len(ms), d - 1),
        "m_expanded_mask": np.array([m["expanded_mask"] for m in ms]),
    }
    for k, f in enumerate(st.factors):
        out[f"factor{k}"] = f
    return out


def blocks_fixture(ref) -> dict:
    b = cases.blocks_inputs()
    out = {}
    for name in ("sym", "psd", "diag312"):
        ev, vec = ref.sym_eig_desc(b[name])
        out[f"eig_{name}_vals"], out[f"eig_{name}_vecs"] = ev, vec
    for name, thr in (("m", 0.5), ("m", 0.0), ("lowrank", 1e-6)):
        l, s, r, disc = ref.small_svd_truncated(b[name], thr)
        key = f"ssvd_{name}_{thr:g}"
        out[key + "_left"], out[key + "_sigma"], out[key + "_right"] = l, s, r
        out[key + "_disc"] = disc
    for name, delta in (("t", 1.0), ("tl", 1e-3)):
        for mode in range(3):
            basis, ev, disc = ref.mode_subspace(b[name], mode, delta)
            key = f"msub_{name}_{mode}"
            out[key + "_basis"], out[key + "_evals"], out[key + "_disc"] = basis, ev, disc
    for mode in range(3):
        a = b["amat"] if mode == 1 else np.ones((2, b["t"].shape[mode]))
        out[f"ttm_t_{mode}"] = ref.ttm(b["t"], mode, a, False)
        out[f"ttm_tT_{mode}"] = ref.ttm(b["t"], mode, a.T.copy(), True)
    # truncation_rank hand cases (test_linalg.cpp:163-174 style)
    tr = []
    for ev, delta in (([4, 1, 0.25, 0.01], np.sqrt(0.3)), ([4, 1, 0.25, 0.01], 0.0),
                      ([4, 1, 0.25, 0.01], 10.0), ([1.0], 0.5), ([5, 5, 5], np.sqrt(5.0))):
        tr.append(ref.truncation_rank(np.array(ev, dtype=float), delta))
    out["trunc_ranks"] = np.array(tr)
    return out


def main():
    ref = po.load_reference()
    for name, fn in cases.STREAM_CASES.items():
        fx = stream_fixture(ref, fn())
        np.savez_compressed(os.path.join(HERE, f"stream_{name}.npz"), **fx)
        print(name, "ranks", fx["core_dims"], "steps", len(fx["m_slice_norm"]),
              "expansions", int(np.count_nonzero(fx["m_expanded_mask"])))
    np.savez_compressed(os.path.join(HERE, "blocks.npz"), **blocks_fixture(ref))
    print("blocks written")


if __name__ == "__main__":
    main()
