"""A/B of the mode-k Gram (SYRK) kernels: DMMA (default) vs TSG_GRAM_FFMA=1.
Run under ncu with -k regex:gram_partial for the kernel times (the wall time
printed here is dominated by the host-side flatten and H2D)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2308_16395_b200.streaming as S
g = np.random.default_rng(3)
shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1:]] or \
    [(384, 384, 640), (200, 200, 1000)]
for dims in shapes:
    t = g.standard_normal(dims)
    S.mode_subspace(t, 0, 0.5 * np.linalg.norm(t))
    t0 = time.perf_counter()
    for _ in range(3):
        b, ev, disc = S.mode_subspace(t, 0, 0.5 * np.linalg.norm(t))
    print(dims, "%.1f ms per mode_subspace (incl. host flatten + H2D of %.2f GB)"
          % ((time.perf_counter() - t0) / 3 * 1e3, t.nbytes / 1e9), "ev0 %.17g" % ev[0])
