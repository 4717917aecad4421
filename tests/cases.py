"""Deterministic parity cases shared by tests/golden/make_golden.py and the tests.

Every case is a function of fixed seeds only (numpy PCG64), so the golden
fixtures generated here from the reference (oracle/_ref) and the inputs the
tests regenerate on the GPU box are byte-identical.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2308_16395_b200 import datagen as dg  # noqa: E402


def _rng(*s):
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(s))))


def flat(t: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64).transpose().ravel())


class StreamCase:
    """init tensor (flat, dims) + list of flat slices + tau."""

    def __init__(self, name, init_flat, init_dims, slices, tau):
        self.name, self.init_flat, self.init_dims = name, init_flat, list(init_dims)
        self.slices, self.tau = slices, tau


def config_case(cfg: dg.StreamConfig, n_slices: int | None = None) -> StreamCase:
    s = dg.make_stream(cfg)
    total = n_slices or cfg.n_slices
    return StreamCase(cfg.name, s.init_numpy(), s.init_dims(),
                      [s.slice_numpy(t) for t in range(cfg.n_init, total)], cfg.tau)


def case_c1() -> StreamCase:
    """BASELINE configs[0] at full size (200 slices of 64x64)."""
    return config_case(dg.CONFIGS["c1"])


def case_growth() -> StreamCase:
    """Config-5 generator at 24^3: spatial ranks grow 3 -> 8 (+1 every 20)."""
    cfg = dg.scaled(dg.CONFIGS["c5"], (24, 24, 24), n_slices=120, n_init=10, name="growth24")
    cfg.growth = (3, 1, 20, 8)
    cfg.spatial_ranks = (8, 8, 8)
    cfg.time_rank = 8
    return config_case(cfg)


def case_c3_small() -> StreamCase:
    """Config-3 generator (geometric core spectrum) at 40^3."""
    cfg = dg.scaled(dg.CONFIGS["c3"], (40, 40, 40), n_slices=30, n_init=5, name="c3_40")
    cfg.spatial_ranks = (12, 12, 12)
    cfg.time_rank = 12
    return config_case(cfg)


def case_thin() -> StreamCase:
    """3-way stream whose mode-1 expansions take the thin route
    (sthosvd.cpp:62-91): rows N_1 = 30 > cols R_0."""
    g = _rng(7, 1)
    n0, n1 = 9, 30
    b0 = np.linalg.qr(g.standard_normal((n0, n0)))[0]
    b1 = np.linalg.qr(g.standard_normal((n1, 12)))[0]
    def sl(t, r):
        c = g.standard_normal((r, r))
        return b0[:, :r] @ c @ b1[:, :r].T
    init = np.stack([sl(t, 2) for t in range(4)], axis=2)
    slices = [flat(sl(t, 2 + (t // 6))) for t in range(30)]
    return StreamCase("thin", flat(init), init.shape, slices, 1e-3)


def case_edges() -> StreamCase:
    """Zero slice, in-span slice, out-of-span slice and a full-rank slice
    (test_streaming.cpp:103-164, 249-302)."""
    g = _rng(11, 2)
    n0, n1, n2 = 6, 5, 4
    basis = np.linalg.qr(g.standard_normal((n0, 3)))[0]
    init = np.zeros((n0, n1, n2))
    for k in range(n2):
        for j in range(n1):
            c0, c1 = g.uniform(-1, 1, 2)
            init[:, j, k] = c0 * basis[:, 0] + c1 * basis[:, 1]
    slices = []
    slices.append(np.zeros((n0, n1)))                                   # zero slice
    slices.append(2.0 * init[:, :, 1] - 0.5 * init[:, :, 3])            # in span
    y = np.zeros((n0, n1))
    for j in range(n1):
        y[:, j] = (g.uniform(-1, 1) + 2.0) * basis[:, 2]                # out of span
    slices.append(y)
    slices.append(g.standard_normal((n0, n1)))                          # full rank
    slices.append(np.zeros((n0, n1)))
    slices.append(g.standard_normal((n0, n1)) * 1e-3)
    return StreamCase("edges", flat(init), init.shape, [flat(s) for s in slices], 1e-6)


def case_random_full() -> StreamCase:
    """Random full-rank data: ranks saturate, many inner-SVD truncations."""
    g = _rng(13, 3)
    init = g.standard_normal((7, 6, 9))
    slices = [flat(g.standard_normal((7, 6))) for _ in range(25)]
    return StreamCase("random_full", flat(init), init.shape, slices, 0.3)


def case_order2() -> StreamCase:
    """Order-2 stream (slices are vectors): only mode 0 plus the ISVD."""
    g = _rng(17, 4)
    u = np.linalg.qr(g.standard_normal((20, 3)))[0]
    init = u @ g.standard_normal((3, 6))
    slices = [flat(u @ g.standard_normal(3) + 1e-3 * g.standard_normal(20)) for _ in range(15)]
    slices[4] = flat(g.standard_normal(20))
    return StreamCase("order2", flat(init), init.shape, slices, 1e-2)


def case_order5() -> StreamCase:
    """5-way stream (slices are 4-way), low-rank plus noise."""
    g = _rng(19, 5)
    dims = (6, 5, 4, 3)
    fac = [np.linalg.qr(g.standard_normal((n, 2)))[0] for n in dims]
    def sl():
        c = g.standard_normal((2, 2, 2, 2))
        x = np.einsum("abcd,ia,jb,kc,ld->ijkl", c, *fac)
        return x + 1e-4 * g.standard_normal(dims)
    init = np.stack([sl() for _ in range(5)], axis=4)
    return StreamCase("order5", flat(init), init.shape, [flat(sl()) for _ in range(12)], 1e-2)


STREAM_CASES = {
    "c1": case_c1,
    "growth24": case_growth,
    "c3_40": case_c3_small,
    "thin": case_thin,
    "edges": case_edges,
    "random_full": case_random_full,
    "order2": case_order2,
    "order5": case_order5,
}


# -------------------------------------------------------- building blocks
def blocks_inputs() -> dict:
    g = _rng(23, 6)
    a = g.standard_normal((9, 9))
    sym = a + a.T
    psd = a @ a.T
    m = g.standard_normal((6, 5))
    lowrank = g.standard_normal((7, 2)) @ g.standard_normal((2, 5))
    t = g.standard_normal((5, 6, 4))
    tl = np.einsum("ia,jb,kc,abc->ijk", g.standard_normal((5, 2)), g.standard_normal((6, 2)),
                   g.standard_normal((4, 2)), g.standard_normal((2, 2, 2)))
    tl = tl + 1e-6 * g.standard_normal(tl.shape)
    amat = g.standard_normal((3, 6))
    return {"sym": sym, "psd": psd, "m": m, "lowrank": lowrank, "t": t, "tl": tl, "amat": amat,
            "diag312": np.diag([3.0, 1.0, 2.0])}


def run_stream(checker_or_state, case: StreamCase, init_fn, update_fn):
    """Drive a stream through init_fn(case) -> handle, update_fn(h, slice)."""
    h = init_fn(case)
    for s in case.slices:
        update_fn(h, s)
    return h
