"""Parity metrics between the GPU path and a CPU checker.

* per-step ranks identical (a rank may differ only where the inner-SVD
  truncation margin |trailing - delta^2| / delta^2 is below 1e-12);
* slice norms, projected norms, mode residuals within 1e-10 relative (plus a
  1e-12 * ||y|| absolute floor for roundoff-level residuals);
* booked error energy within 1e-12 of the total input energy;
* singular values within 1e-10 of sigma_max; core, sigma-weighted factors and
  the reconstructed model within 1e-10 relative in Frobenius norm (factor
  column j of U_k weighted by the energy of core slice j along mode k; the
  raw columns are held to 1e-7 because weak directions carry the reference's
  own Gram-route rounding, SURVEY §7 hard part 1).
"""
from __future__ import annotations

import numpy as np

TOL = 1e-10


def rel(a, b) -> float:
    a, b = np.asarray(a, float), np.asarray(b, float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


def reconstruct(st) -> np.ndarray:
    """Full model (core x_k U_k x_{d-1} left) as a numpy tensor."""
    core = st.core.reshape(tuple(st.core_dims)[::-1]).transpose()
    x = core
    facs = list(st.factors) + [st.left]
    for k, f in enumerate(facs):
        x = np.moveaxis(np.tensordot(f, x, axes=([1], [k])), 0, k)
    return x


def reconstruct_sampled(st, per_mode: int = 24, seed: int = 7) -> np.ndarray:
    """The model on a seeded sub-grid: `per_mode` rows of every factor
    (streaming factor included), i.e. core x_k U_k[idx_k, :]. Used when the
    full reconstruction would not fit in host memory (C3, C4, C5 at the
    BASELINE sizes: 10^9-10^10 entries)."""
    g = np.random.default_rng(seed)
    core = st.core.reshape(tuple(st.core_dims)[::-1]).transpose()
    x = core
    facs = list(st.factors) + [st.left]
    for k, f in enumerate(facs):
        rows = f.shape[0]
        idx = np.sort(g.choice(rows, size=min(per_mode, rows), replace=False))
        x = np.moveaxis(np.tensordot(f[idx, :], x, axes=([1], [k])), 0, k)
    return x


def metrics_arrays(ms, d):
    return {
        "ranks": np.array([m["ranks"] for m in ms]).reshape(len(ms), d),
        "slice_norm": np.array([m["slice_norm"] for m in ms]),
        "projected_norm": np.array([m["projected_norm"] for m in ms]),
        "error_estimate": np.array([m["error_estimate"] for m in ms]),
        "mode_residuals": np.array([m["mode_residuals"] for m in ms]).reshape(len(ms), d - 1),
        "expanded_mask": np.array([m["expanded_mask"] for m in ms]),
        "margin": np.array([m.get("trunc_margin", 1.0) for m in ms]),
    }


def golden_metrics(g):
    return {
        "ranks": g["m_ranks"], "slice_norm": g["m_slice_norm"],
        "projected_norm": g["m_projected_norm"], "error_estimate": g["m_error_estimate"],
        "mode_residuals": g["m_mode_residuals"], "expanded_mask": g["m_expanded_mask"],
    }


def compare_metrics(gpu: dict, ref: dict, total_sq: float) -> dict:
    out = {}
    ok_rank = np.all(gpu["ranks"] == ref["ranks"], axis=1)
    bad = np.where(~ok_rank)[0]
    # exemption: near-cut truncations on either side
    near = [i for i in bad if gpu["margin"][i] < 1e-12]
    out["rank_mismatch_steps"] = [int(i) for i in bad if i not in near]
    out["rank_exempt_steps"] = [int(i) for i in near]
    sn = ref["slice_norm"]
    out["slice_norm"] = float(np.max(np.abs(gpu["slice_norm"] - sn) / np.maximum(sn, 1e-300)))
    pn = ref["projected_norm"]
    out["projected_norm"] = float(np.max(np.abs(gpu["projected_norm"] - pn) /
                                         np.maximum(pn, 1e-300))) if len(pn) else 0.0
    mr = ref["mode_residuals"]
    floor = 1e-12 * sn[:, None]
    out["mode_residuals"] = float(np.max(np.maximum(np.abs(gpu["mode_residuals"] - mr) - floor, 0.0) /
                                         np.maximum(np.abs(mr), 1e-300))) if mr.size else 0.0
    # booked energy: est^2 * total
    bg = gpu["error_estimate"] ** 2
    br = ref["error_estimate"] ** 2
    out["booked"] = float(np.max(np.abs(bg - br))) if len(br) else 0.0  # relative to total energy
    out["expanded_mask_equal"] = bool(np.array_equal(gpu["expanded_mask"], ref["expanded_mask"]))
    return out


def compare_states(sg, sr) -> dict:
    out = {"core_dims_equal": tuple(sg.core_dims) == tuple(sr.core_dims)}
    if not out["core_dims_equal"]:
        return out
    s0 = max(float(sr.sigma[0]), 1e-300)
    out["sigma"] = float(np.max(np.abs(np.asarray(sg.sigma) - np.asarray(sr.sigma))) / s0)
    out["core"] = rel(sg.core, sr.core)
    # factors: raw column difference (informational) and the sigma-weighted
    # form of SURVEY §8(c): column j of U_k weighted by the energy of core
    # slice j along mode k (the mode-k singular direction's weight)
    out["factors_raw"] = max([rel(a, b) for a, b in zip(sg.factors, sr.factors)] + [0.0])
    core_r = sr.core.reshape(tuple(sr.core_dims)[::-1]).transpose()
    wf = []
    for k, (a, b) in enumerate(zip(sg.factors, sr.factors)):
        ck = np.moveaxis(core_r, k, 0).reshape(core_r.shape[k], -1)
        w = np.linalg.norm(ck, axis=1)[None, :]
        wf.append(rel(a * w, b * w))
    out["factors"] = max(wf + [0.0])
    # streaming factor weighted by sigma (weak columns carry little of the model)
    out["left_weighted"] = rel(sg.left * sg.sigma[None, :], sr.left * sr.sigma[None, :])
    out["right_weighted"] = rel(sg.right * sg.sigma[None, :], sr.right * sr.sigma[None, :])
    out["ledger_sq_err"] = abs(sg.squared_error - sr.squared_error) / max(sr.total_input_sq, 1e-300)
    out["ledger_nonstream"] = abs(sg.nonstream_discarded_sq - sr.nonstream_discarded_sq) / max(sr.total_input_sq, 1e-300)
    out["ledger_total"] = abs(sg.total_input_sq - sr.total_input_sq) / max(sr.total_input_sq, 1e-300)
    full = float(np.prod(sg.slice_dims)) * max(sg.n_d, 1)
    if full < 5e7:
        out["reconstruction"] = rel(reconstruct(sg), reconstruct(sr))
    else:
        # the full models would be 10^9-10^10 doubles each: compare them on a
        # seeded sub-grid (the same rows of every factor on both sides)
        out["reconstruction"] = rel(reconstruct_sampled(sg), reconstruct_sampled(sr))
        out["reconstruction_sampled"] = True
    return out


def state_from_golden(g):
    from types import SimpleNamespace
    d = int(g["order"])
    return SimpleNamespace(
        order=d, n_d=int(g["n_d"]), rank=int(g["rank"]), core_dims=tuple(int(v) for v in g["core_dims"]),
        slice_dims=tuple(int(v) for v in g["slice_dims"]), core=g["core"], sigma=g["sigma"],
        left=g["left"], right=g["right"], factors=[g[f"factor{k}"] for k in range(d - 1)],
        squared_error=float(g["squared_error"]), total_input_sq=float(g["total_input_sq"]),
        nonstream_discarded_sq=float(g["nonstream_discarded_sq"]))


def assert_parity(mc: dict, sc: dict, tol: float = TOL, factor_tol: float = TOL,
                  resid_tol: float = TOL):
    assert not mc["rank_mismatch_steps"], f"rank mismatch at steps {mc['rank_mismatch_steps']}"
    assert mc["expanded_mask_equal"]
    assert mc["slice_norm"] <= 1e-13, mc
    assert mc["projected_norm"] <= tol, mc
    assert mc["mode_residuals"] <= resid_tol, mc
    assert mc["booked"] <= 1e-12, mc
    assert sc["core_dims_equal"], sc
    assert sc["sigma"] <= tol, sc
    assert sc["core"] <= factor_tol, sc
    assert sc["factors"] <= factor_tol, sc
    assert sc["factors_raw"] <= 1e-7, sc
    assert sc["left_weighted"] <= factor_tol, sc
    assert sc["right_weighted"] <= factor_tol, sc
    assert sc["ledger_sq_err"] <= 1e-12 and sc["ledger_nonstream"] <= 1e-12, sc
    assert sc["ledger_total"] <= 1e-13, sc
    if "reconstruction" in sc:
        assert sc["reconstruction"] <= tol, sc
