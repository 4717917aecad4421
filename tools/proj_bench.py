"""Time the fused projection kernel alone on C2/C3-shaped inputs."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
L = S.load_library()
L.tsg_debug_project.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
dev = torch.device("cuda", 0)
for (left, n, right, R) in [(1, 200, 40000, 10), (10, 200, 200, 10), (100, 200, 1, 10),
                            (1, 512, 262144, 32), (1, 256, 65536, 12)]:
    x = torch.randn(left * n * right, dtype=torch.float64, device=dev)
    u = torch.linalg.qr(torch.randn(n, R, dtype=torch.float64, device=dev))[0].t().contiguous().t().contiguous()
    u = u.t().contiguous().view(-1)  # column-major n x R
    p = torch.empty(left * R * right, dtype=torch.float64, device=dev)
    res = []
    for flags in (0, 1, 2, 3):
        ms = C.c_double()
        rc = L.tsg_debug_project(x.data_ptr(), left, n, right, u.data_ptr(), R, p.data_ptr(), flags, 20, C.byref(ms))
        res.append(f"f{flags}={ms.value*1e3:.1f}us")
    gb = 8 * (left * n * right) / 1e9
    print(f"left={left} n={n} right={right} R={R} ({gb*1e3:.0f} MB):", " ".join(res), f"hbm-floor={gb/6.5e3*1e6:.1f}us")
