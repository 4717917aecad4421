"""Reference API pieces beyond the per-slice update, on the B200 path:

* ISVDOptions::reorthogonalize_every (isvd.hpp:62-67, isvd.cpp:243-248):
  MGS of the streaming and right factors every K insertions, against the
  pinned C restatement (bit-identical to the reference with the option on,
  tests/test_oracle.py) and the reference's own property test
  (test_isvd.cpp:408-428: a long lossy stream stays orthonormal);
* TUCKCKPT v1 checkpoints (io.cpp:268-423): bit-exact resume
  (test_io.cpp:209-247), files read by the reference's load_checkpoint and
  written by its save_checkpoint, and the loader's error behaviour.
"""
import os

import numpy as np
import pytest

import cases
import parity as P

pytestmark = pytest.mark.gpu

S = pytest.importorskip("paper_2308_16395_b200.streaming")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu(case, k=0, asynchronous=False, n=None):
    st = S.StreamingState(asynchronous=asynchronous, reorthogonalize_every=k)
    st.init_flat(case.init_flat, case.init_dims, case.tau)
    for s in case.slices[:n]:
        st.stream_update(s)
    st.synchronize()
    return st


def _checker(chk, case, k=0, n=None):
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    h = chk.stream_init(x, case.tau)
    if k:
        h.set_reorthogonalize_every(k)
    for s in case.slices[:n]:
        h.update_flat(s)
    return h


@pytest.mark.parametrize("name,k,asynchronous", [
    ("growth", 3, False), ("growth", 3, True), ("growth", 16, True), ("c3_small", 5, True)])
def test_reorthogonalization_vs_oracle(oracle, name, k, asynchronous):
    case = {"growth": cases.case_growth, "c3_small": cases.case_c3_small}[name]()
    st = _gpu(case, k, asynchronous)
    ho = _checker(oracle, case, k)
    sg, so = st.export(), ho.export()
    mc = P.compare_metrics(P.metrics_arrays(st.metrics(), sg.order),
                           P.metrics_arrays(ho.metrics(), so.order), so.total_input_sq)
    sc = P.compare_states(sg, so)
    print(name, k, mc, sc)
    P.assert_parity(mc, sc)
    assert np.abs(sg.left.T @ sg.left - np.eye(sg.rank)).max() <= 1e-12


def test_reorthogonalization_long_lossy_stream(oracle):
    """test_isvd.cpp:408-428 in streaming form: 300 lossy random slices
    (tau = 0.3), K = 16: both factors stay orthonormal to 1e-10, and the
    state matches the checker."""
    g = np.random.default_rng(41)
    dims = (6, 4)
    init = g.uniform(-1, 1, dims + (4,))
    slices = [cases.flat(g.uniform(-1, 1, dims)) for _ in range(300)]
    case = cases.StreamCase("lossy", cases.flat(init), init.shape, slices, 0.3)
    st = _gpu(case, 16, True)
    ho = _checker(oracle, case, 16)
    sg, so = st.export(), ho.export()
    assert np.abs(sg.left.T @ sg.left - np.eye(sg.rank)).max() <= 1e-10
    assert np.abs(sg.right.T @ sg.right - np.eye(sg.rank)).max() <= 1e-10
    mc = P.compare_metrics(P.metrics_arrays(st.metrics(), sg.order),
                           P.metrics_arrays(ho.metrics(), so.order), so.total_input_sq)
    P.assert_parity(mc, P.compare_states(sg, so))


def _fields_equal(a, b):
    assert a.core_dims == b.core_dims and a.n_d == b.n_d
    for f in ("core", "sigma", "left", "right"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    for fa, fb in zip(a.factors, b.factors):
        np.testing.assert_array_equal(fa, fb)
    assert (a.squared_error, a.total_input_sq, a.nonstream_discarded_sq) == \
        (b.squared_error, b.total_input_sq, b.nonstream_discarded_sq)


def test_checkpoint_resume_bitexact(tmp_path):
    """save -> load -> continue == uninterrupted (test_io.cpp:209-247)."""
    case = cases.case_growth()
    full = _gpu(case).export()
    half = len(case.slices) // 2
    st = _gpu(case, n=half)
    path = str(tmp_path / "state.ckpt")
    st.save_checkpoint(path)
    assert not os.path.exists(path + ".tmp")
    st2 = S.load_checkpoint(path)
    _fields_equal(st2.export(), st.export())
    for s in case.slices[half:]:
        st2.stream_update(s)
    _fields_equal(st2.export(), full)


def test_checkpoint_interoperates_with_reference(reference, tmp_path):
    """Our file is read by the reference's load_checkpoint + from_checkpoint
    (identical state), its save_checkpoint file is read by ours (identical
    bytes after a round trip), and both continue identically."""
    case = cases.case_c3_small()
    st = _gpu(case, n=10)
    ours = str(tmp_path / "ours.ckpt")
    st.save_checkpoint(ours)
    h = reference.load_checkpoint(ours)
    _fields_equal(h.export(), st.export())
    theirs = str(tmp_path / "theirs.ckpt")
    h.save_checkpoint(theirs)
    assert open(theirs, "rb").read() == open(ours, "rb").read()
    st2 = S.load_checkpoint(theirs)
    for s in case.slices[10:]:
        st2.stream_update(s)
        h.update_flat(s)
    sg, so = st2.export(), h.export()
    mc = P.compare_metrics(P.metrics_arrays(st2.metrics(), sg.order),
                           P.metrics_arrays(h.metrics(), so.order), so.total_input_sq)
    P.assert_parity(mc, P.compare_states(sg, so))


def test_checkpoint_loader_errors(tmp_path):
    """load_checkpoint's validation (io.cpp:326-412) and from_checkpoint's
    refusal of batch models (io.cpp:414-418); a state whose core drifted
    from v x diag(s) is refused at assembly (streaming.cpp:55-62)."""
    case = cases.case_growth()
    st = _gpu(case, n=5)
    good = tmp_path / "good.ckpt"
    st.save_checkpoint(str(good))
    blob = good.read_bytes()
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"XUCKCKPT" + blob[8:])
    with pytest.raises(S.IoError, match="bad magic"):
        S.load_checkpoint(str(bad))
    bad.write_bytes(blob[:8] + (2).to_bytes(4, "little") + blob[12:])
    with pytest.raises(S.IoError, match="bad version"):
        S.load_checkpoint(str(bad))
    bad.write_bytes(blob[:-40])
    with pytest.raises(S.IoError, match="truncated"):
        S.load_checkpoint(str(bad))
    with pytest.raises(S.IoError):
        S.load_checkpoint(str(tmp_path / "missing.ckpt"))
    d = st.query()["order"]
    flag_at = 8 + 4 + 4 + 8 * d * 2 + 8 + 8 * d
    bad.write_bytes(blob[:flag_at] + (0).to_bytes(4, "little") + blob[flag_at + 4:])
    with pytest.raises(S.InvalidArgument):
        S.load_checkpoint(str(bad))
    core_at = flag_at + 4
    raw = bytearray(blob)
    v = np.frombuffer(bytes(raw[core_at:core_at + 8]), dtype="<f8")[0]
    raw[core_at:core_at + 8] = np.array([v * (1 + 1e-4) + 1e-3], dtype="<f8").tobytes()
    bad.write_bytes(bytes(raw))
    with pytest.raises(S.CouplingDrift):
        S.load_checkpoint(str(bad))


@pytest.mark.parametrize("name", ["growth24", "c3_40", "order5", "order2"])
def test_add_row_composes_stream_update(oracle, name):
    """tsg_add_row (add_row, isvd.hpp:110-111 / isvd.cpp:163-250, plus the core
    rotation of streaming.cpp:199-222): one stream_update equals
    process_nonstreaming_mode for every mode followed by add_row with
    delta = tau ||y|| / sqrt(d) (the reference's own decomposition,
    streaming.cpp:187-200). The composed state matches the one-call state to
    rounding and the CPU checker to the parity bounds; AddRowResult's fields
    follow the ranks."""
    case = cases.STREAM_CASES[name]()
    n = min(len(case.slices), 14)
    one = _gpu(case, n=n)
    st = S.StreamingState()
    st.init_flat(case.init_flat, case.init_dims, case.tau)
    dims = tuple(case.init_dims[:-1])
    d = len(case.init_dims)
    for y in case.slices[:n]:
        t = y.reshape(dims[::-1]).transpose()
        nrm = float(np.linalg.norm(y))
        delta = case.tau * nrm / np.sqrt(d)
        cur = t
        for k in range(d - 1):
            _, cur = st.process_nonstreaming_mode(cur, k, delta)
        r_before = st.query()["rank"]
        res = st.add_row(cur, delta, slice_norm_sq=nrm * nrm)
        assert res["r_old"] == r_before and res["r_new"] == st.query()["rank"]
        assert res["r_new"] <= res["r_old"] + 1 and res["added_error_sq"] >= 0.0
    a, b = st.export(), one.export()
    assert a.core_dims == b.core_dims and a.n_d == b.n_d
    sc = P.compare_states(a, b)
    print(name, "composed vs one call", sc)
    assert sc["core"] <= 1e-11 and sc["sigma"] <= 1e-12 and sc["factors"] <= 1e-11
    assert sc["ledger_sq_err"] <= 1e-13 and sc["ledger_nonstream"] <= 1e-13 and sc["ledger_total"] <= 1e-14
    so = _checker(oracle, case, n=n).export()
    P.assert_parity({"rank_mismatch_steps": [], "expanded_mask_equal": True, "slice_norm": 0.0,
                     "projected_norm": 0.0, "mode_residuals": 0.0, "booked": 0.0},
                    P.compare_states(a, so))
    with pytest.raises(S.InvalidArgument):
        st.add_row(np.zeros(int(np.prod(a.core_dims[:-1]))), -1.0)
