"""Check the fused projection (P = U^T X_(k), residual norms) against torch fp64
for a sweep of (left, N, right, R) shapes, through tsg_debug_project."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
L = S.load_library()
L.tsg_debug_project.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
dev = torch.device("cuda", 0)
shapes = [(1, 320, 200000, 22), (1, 320, 20000, 22), (7, 96, 96, 20), (1, 96, 2000, 20), (1, 320, 20000, 35),
          (1, 320, 20000, 12), (1, 384, 20000, 41), (1, 384, 20000, 36), (40, 384, 300, 41), (1, 384, 5000, 63),
          (63, 384, 100, 98), (1, 512, 3000, 32), (1, 200, 4000, 10), (7, 96, 96, 20), (1, 256, 3000, 36),
          (1, 48, 2000, 38)]
bad = 0
for (left, n, right, R) in shapes:
    g = torch.Generator(device=dev); g.manual_seed(1)
    x = torch.randn(right, n, left, dtype=torch.float64, device=dev, generator=g)  # x[r, i, l] = X[l + i*left + r*left*n]
    u = torch.linalg.qr(torch.randn(n, R, dtype=torch.float64, device=dev, generator=g))[0]
    ucm = u.t().contiguous()  # column-major n x R == row-major R x n
    p = torch.zeros(right * R * left, dtype=torch.float64, device=dev)
    ms = C.c_double()
    rc = L.tsg_debug_project(x.data_ptr(), left, n, right, ucm.data_ptr(), R, p.data_ptr(), 0, 1, C.byref(ms))
    ref = torch.einsum("ir,bil->brl", u, x)  # P[l + j*left + r*left*R]
    got = p.view(right, R, left)
    err = (got - ref).norm() / ref.norm()
    ok = rc == 0 and err < 1e-12
    bad += not ok
    msg = "" if rc == 0 else L.tsg_last_error(None).decode()
    print(f"left={left} N={n} right={right} R={R}: rc={rc} relerr={err:.2e} {'ok' if ok else 'BAD'} {ms.value*1e3:.1f}us {msg}")
print("bad", bad)
