"""mode_subspace (device) vs numpy eigh on large shapes."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_16395_b200.streaming as S
g = np.random.default_rng(3)
for dims in [(256, 256, 16), (320, 320, 16), (320, 64, 16), (288, 100, 8), (384, 50, 16)]:
    r = 30
    facs = [np.linalg.qr(g.standard_normal((n, min(r, n))))[0] for n in dims]
    c = g.standard_normal(tuple(f.shape[1] for f in facs))
    t = np.einsum("abc,ia,jb,kc->ijk", c, *facs) + 1e-3 * g.standard_normal(dims)
    delta = 1e-2 * np.linalg.norm(t)
    basis, ev, disc = S.mode_subspace(t, 0, delta)
    a = t.reshape(dims[0], -1, order="F")
    w, v = np.linalg.eigh(a @ a.T)
    w, v = w[::-1], v[:, ::-1]
    k = basis.shape[1]
    orth = np.max(np.abs(basis.T @ basis - np.eye(k)))
    sub = np.linalg.norm(basis @ (basis.T @ v[:, :k]) - v[:, :k])
    print(dims, "rank", k, "orth %.1e" % orth, "subspace err %.1e" % sub, "ev rel %.1e" % (np.max(np.abs(ev[:k] - w[:k])) / w[0]))
