"""Time the device symmetric eigensolver (sym_eig_desc) on random Gram-like
matrices (env TSG_COOP_EIG_MIN selects the single-CTA / cooperative path)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_16395_b200.streaming as S
g = np.random.default_rng(1)
for n in (96, 128, 200, 256, 300, 384, 440):
    a = g.standard_normal((n, 3 * n))
    G = a @ a.T
    S.sym_eig_desc(G)  # warm
    t0 = time.perf_counter()
    for _ in range(3):
        ev, vec = S.sym_eig_desc(G)
    dt = (time.perf_counter() - t0) / 3
    w = np.linalg.eigvalsh(G)[::-1]
    import hashlib
    h = hashlib.sha1(ev.tobytes() + vec.tobytes()).hexdigest()[:12]
    print(n, "%.2f ms" % (dt * 1e3), "ev err %.1e" % (np.max(np.abs(ev - w)) / w[0]), h)
