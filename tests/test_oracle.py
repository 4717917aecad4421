"""CPU tests: pin the C restatement (oracle/liboracle.so) against the
reference's own outputs — the golden fixtures made by oracle/_ref — and,
where the reference build is present, against the reference directly."""
import numpy as np
import pytest

import cases
import py_oracle as po
from golden.make_golden import input_digest

STATE_ARRAYS = ("core", "sigma", "left", "right")
METRIC_ARRAYS = ("m_ranks", "m_slice_norm", "m_projected_norm", "m_error_estimate",
                 "m_mode_residuals", "m_expanded_mask")


def run_checker(chk, case):
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    h = chk.stream_init(x, case.tau)
    for s in case.slices:
        h.update_flat(s)
    return h


@pytest.mark.parametrize("name", sorted(cases.STREAM_CASES))
def test_oracle_bitexact_vs_golden(oracle, golden, name):
    case = cases.STREAM_CASES[name]()
    g = golden("stream_" + name)
    assert str(g["digest"]) == input_digest(case), "input generator drifted"
    h = run_checker(oracle, case)
    st = h.export()
    assert tuple(st.core_dims) == tuple(g["core_dims"])
    assert st.n_d == g["n_d"] and st.rank == g["rank"] and st.insertions == g["insertions"]
    for k in STATE_ARRAYS:
        np.testing.assert_array_equal(getattr(st, k), g[k], err_msg=k)
    for k, f in enumerate(st.factors):
        np.testing.assert_array_equal(f, g[f"factor{k}"])
    for k in ("squared_error", "total_input_sq", "nonstream_discarded_sq"):
        assert getattr(st, k) == g[k], k
    ms = h.metrics()
    d = st.order
    got = {
        "m_ranks": np.array([m["ranks"] for m in ms]).reshape(len(ms), d),
        "m_slice_norm": np.array([m["slice_norm"] for m in ms]),
        "m_projected_norm": np.array([m["projected_norm"] for m in ms]),
        "m_error_estimate": np.array([m["error_estimate"] for m in ms]),
        "m_mode_residuals": np.array([m["mode_residuals"] for m in ms]).reshape(len(ms), d - 1),
        "m_expanded_mask": np.array([m["expanded_mask"] for m in ms]),
    }
    for k in METRIC_ARRAYS:
        np.testing.assert_array_equal(got[k], g[k], err_msg=k)


def test_oracle_blocks_vs_golden(oracle, golden):
    g = golden("blocks")
    b = cases.blocks_inputs()
    for name in ("sym", "psd", "diag312"):
        ev, vec = oracle.sym_eig_desc(b[name])
        np.testing.assert_array_equal(ev, g[f"eig_{name}_vals"])
        np.testing.assert_array_equal(vec, g[f"eig_{name}_vecs"])
    for name, thr in (("m", 0.5), ("m", 0.0), ("lowrank", 1e-6)):
        l, s, r, disc = oracle.small_svd_truncated(b[name], thr)
        key = f"ssvd_{name}_{thr:g}"
        np.testing.assert_array_equal(l, g[key + "_left"])
        np.testing.assert_array_equal(s, g[key + "_sigma"])
        np.testing.assert_array_equal(r, g[key + "_right"])
        assert disc == g[key + "_disc"]
    for name, delta in (("t", 1.0), ("tl", 1e-3)):
        for mode in range(3):
            basis, ev, disc = oracle.mode_subspace(b[name], mode, delta)
            key = f"msub_{name}_{mode}"
            np.testing.assert_array_equal(basis, g[key + "_basis"])
            np.testing.assert_array_equal(ev, g[key + "_evals"])
            assert disc == g[key + "_disc"]
    for mode in range(3):
        a = b["amat"] if mode == 1 else np.ones((2, b["t"].shape[mode]))
        np.testing.assert_array_equal(oracle.ttm(b["t"], mode, a, False), g[f"ttm_t_{mode}"])
        np.testing.assert_array_equal(oracle.ttm(b["t"], mode, a.T.copy(), True), g[f"ttm_tT_{mode}"])
    tr = []
    for ev, delta in (([4, 1, 0.25, 0.01], np.sqrt(0.3)), ([4, 1, 0.25, 0.01], 0.0),
                      ([4, 1, 0.25, 0.01], 10.0), ([1.0], 0.5), ([5, 5, 5], np.sqrt(5.0))):
        tr.append(oracle.truncation_rank(np.array(ev, dtype=float), delta))
    np.testing.assert_array_equal(np.array(tr), g["trunc_ranks"])


def test_known_answers(oracle):
    # diag(3,1,2): descending eigenvalues, sign rule (test_linalg.cpp:69-82)
    ev, vec = oracle.sym_eig_desc(np.diag([3.0, 1.0, 2.0]))
    np.testing.assert_array_equal(ev, [3.0, 2.0, 1.0])
    np.testing.assert_array_equal(vec, np.eye(3)[:, [0, 2, 1]])
    # truncation hand case (test_linalg.cpp:163-174)
    assert oracle.truncation_rank(np.array([4, 1, 0.25, 0.01]), np.sqrt(0.3)) == 2
    assert oracle.truncation_rank(np.array([4, 1, 0.25, 0.01]), 100.0) == 1  # clamped >= 1
    with pytest.raises(po.InvalidArgument):
        oracle.truncation_rank(np.array([1.0, 2.0]), 0.1)
    # small_svd on diag(3, 1e-9), threshold 1e-6 -> rank 1 (test_linalg.cpp:196-212)
    l, s, r, disc = oracle.small_svd_truncated(np.diag([3.0, 1e-9]), 1e-6)
    assert len(s) == 1 and s[0] == pytest.approx(3.0, rel=1e-15)
    assert disc == pytest.approx(1e-18, rel=1e-6)
    # ttm with an all-ones row (test_tensor_core.cpp:118-127)
    t = np.arange(1, 9, dtype=float).reshape(2, 2, 2, order="F")
    out = oracle.ttm(t, 0, np.ones((1, 2)))
    np.testing.assert_array_equal(out.ravel(order="F"), [3, 7, 11, 15])


def test_error_behaviour(oracle):
    with pytest.raises(po.InvalidArgument):
        oracle.stream_init(np.zeros((5, 4, 3)), 0.5)          # zero batch
    with pytest.raises(po.InvalidArgument):
        oracle.stream_init(np.ones(6), 0.5)                    # order 1
    ok = np.random.default_rng(3).standard_normal((4, 5, 2))
    for tau in (0.0, 1.0):
        with pytest.raises(po.InvalidArgument):
            oracle.stream_init(ok, tau)


def test_oracle_vs_reference_random(oracle, reference):
    """Random streams with expansions: the restatement is bit-identical to
    the reference build (same op order, no FMA contraction)."""
    rng = np.random.default_rng(2026)
    for trial in range(6):
        dims = [int(v) for v in rng.integers(3, 10, size=3 + trial % 2)]
        r = 2
        x = rng.standard_normal(dims[:-1] + [dims[-1]])
        # low-rank init to force expansions later
        fac = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n in dims[:-1]]
        core = rng.standard_normal([r] * (len(dims) - 1) + [dims[-1]])
        x = core
        for k, f in enumerate(fac):
            x = np.moveaxis(np.tensordot(f, x, axes=([1], [k])), 0, k)
        tau = [1e-2, 1e-3, 0.1, 1e-4, 0.05, 0.2][trial]
        ho, hr = oracle.stream_init(x, tau), reference.stream_init(x, tau)
        for t in range(20):
            y = rng.standard_normal(dims[:-1]) * (0.0 if t == 7 else 1.0)
            ho.stream_update(y)
            hr.stream_update(y)
        so, sr = ho.export(), hr.export()
        assert so.core_dims == sr.core_dims
        for k in STATE_ARRAYS:
            np.testing.assert_array_equal(getattr(so, k), getattr(sr, k))
        assert ho.metrics() == hr.metrics()


def test_process_mode_vs_reference(oracle, reference):
    case = cases.case_edges()
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    y = case.slices[2].reshape(case.init_dims[:-1][::-1]).transpose()
    ho, hr = oracle.stream_init(x, case.tau), reference.stream_init(x, case.tau)
    ro, yo = ho.process_nonstreaming_mode(y, 0, 1e-6 * np.linalg.norm(y))
    rr, yr = hr.process_nonstreaming_mode(y, 0, 1e-6 * np.linalg.norm(y))
    assert ro == rr
    np.testing.assert_array_equal(yo, yr)
    np.testing.assert_array_equal(ho.export().factors[0], hr.export().factors[0])


def test_config4_generator_layout_and_noise_rule():
    """The config-4 generator: colexicographic layout, bounded tanh values,
    the reference's per-slice noise rule ||N|| = eta ||X|| (datagen.cpp:90-101)
    and a torch synthesis equal to the numpy one up to the noise."""
    from paper_2308_16395_b200 import datagen as dg
    cfg = dg.scaled(dg.CONFIGS["c4"], (12, 10, 8, 4), n_slices=4, n_init=2)
    s = dg.make_stream(cfg)
    clean = s.clean_slice_numpy(1)
    assert clean.shape == (12, 10, 8, 4) and np.all(np.abs(clean) < 1.0)
    flat = s.slice_numpy(1)
    t = flat.reshape((4, 8, 10, 12)).transpose()
    noise = t - clean
    assert np.linalg.norm(noise) == pytest.approx(cfg.eta * np.linalg.norm(clean), rel=1e-9)
    torch = pytest.importorskip("torch")
    b = s.slice_torch(1, "cpu").numpy()
    assert np.linalg.norm(b - flat) <= 3 * cfg.eta * np.linalg.norm(flat)
    assert s.init_dims() == [12, 10, 8, 4, 2]


def test_restatement_matches_reference_with_reorthogonalization(reference, oracle):
    """ISVDOptions::reorthogonalize_every (isvd.hpp:62-67, isvd.cpp:243-248):
    the C restatement stays bit-identical to the reference with the periodic
    MGS of both factors enabled."""
    import cases
    case = cases.case_growth()
    out = []
    for chk in (reference, oracle):
        x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
        h = chk.stream_init(x, case.tau)
        h.set_reorthogonalize_every(3)
        for s in case.slices[:40]:
            h.update_flat(s)
        out.append(h.export())
    a, b = out
    assert a.core_dims == b.core_dims
    for f in ("core", "sigma", "left", "right"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    assert np.abs(a.left.T @ a.left - np.eye(a.rank)).max() <= 1e-12
