"""Launch the mode-0 projection kernel (C2 or C3 shape) a few times on device
buffers; for ncu captures of proj0_tma_kernel alone."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2308_16395_b200.streaming as S
L = S.load_library()
L.tsg_debug_project.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
shape = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 64: TMA kernel streams only
n, right, R = {"c2": (200, 40000, 10), "c3": (512, 262144, 32), "c5": (256, 65536, 8),
               "c5l": (256, 65536, 36)}[shape]
dev = torch.device("cuda", 0)
x = torch.randn(n * right, dtype=torch.float64, device=dev)
u = torch.linalg.qr(torch.randn(n, R, dtype=torch.float64, device=dev))[0]
u = u.t().contiguous().view(-1)  # column-major n x R
p = torch.empty(R * right, dtype=torch.float64, device=dev)
ms = C.c_double()
rc = L.tsg_debug_project(x.data_ptr(), 1, n, right, u.data_ptr(), R, p.data_ptr(), flags, reps, C.byref(ms))
gb = 8 * n * right / 1e9
print(f"{shape}: rc={rc} {ms.value*1e3:.1f} us/launch, {gb/ms.value*1e3:.0f} GB/s, {4*R*n*right/ms.value/1e9:.1f} TF/s")
