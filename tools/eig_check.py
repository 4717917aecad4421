"""Check the device eigensolver (single-CTA and cooperative paths) against numpy."""
import sys, os, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_16395_b200.streaming as S
for n in (64, 100, 256, 512):
    g = np.random.default_rng(n).standard_normal((n, 3 * n))
    a = g @ g.T
    t0 = time.time()
    ev, vec = S.sym_eig_desc(a)
    dt = time.time() - t0
    ref = np.sort(np.linalg.eigvalsh(a))[::-1]
    res = np.linalg.norm(a @ vec - vec * ev[None, :]) / np.linalg.norm(a)
    orth = np.max(np.abs(vec.T @ vec - np.eye(n)))
    print(n, f"{dt*1e3:.1f} ms", "eval err", np.max(np.abs(ev - ref)) / ref[0], "resid", res, "orth", orth)
