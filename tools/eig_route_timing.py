"""Time mode_subspace's eigensolve routes on Gram-like inputs: the tridiagonal
route (default for n >= 96) against the cooperative Jacobi (TSG_EIG_TRI=0),
through tsg_mode_subspace on a host tensor (times include the H2D copy and
the Gram, identical for both routes). Usage: eig_route_timing.py"""
import os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2308_16395_b200.streaming as S
    g = np.random.default_rng(1)
    for n in (96, 128, 200, 256, 384, 512):
        u = np.linalg.qr(g.standard_normal((n, n)))[0]
        sv = np.concatenate([np.linspace(10, 3, 12), 1e-4 * (1 + g.random(n - 12))])
        a = (u * sv[None, :]) @ np.linalg.qr(g.standard_normal((2 * n, n)))[0].T
        t = a.reshape(n, 2 * n, 1)
        delta = float(np.sqrt(np.sum(sv[12:] ** 2) * 1.5))
        S.mode_subspace(t, 0, delta)
        t0 = time.perf_counter()
        for _ in range(5):
            basis, ev, disc = S.mode_subspace(t, 0, delta)
        dt = (time.perf_counter() - t0) / 5
        w = np.linalg.eigvalsh(a @ a.T)[::-1]
        print(f"  n {n:4d}: {dt * 1e3:7.2f} ms per mode_subspace, rank {basis.shape[1]}, "
              f"eigenvalue err {np.max(np.abs(ev - w.clip(min=0))) / w[0]:.1e}", flush=True)
else:
    for env, label in ((None, "tridiagonal route"), ("0", "cooperative Jacobi (TSG_EIG_TRI=0)")):
        e = dict(os.environ)
        if env is not None:
            e["TSG_EIG_TRI"] = env
        print(label, flush=True)
        subprocess.run([sys.executable, os.path.abspath(__file__), "child"], env=e, check=False)
