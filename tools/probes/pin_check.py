"""Is a large torch pin_memory() buffer page-locked for the CUDA driver?"""
import ctypes, sys, time
import torch
rt = ctypes.CDLL("libcudart.so.12") if len(sys.argv) < 2 else ctypes.CDLL(sys.argv[1])
class Attr(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("device", ctypes.c_int), ("devicePointer", ctypes.c_void_p),
                ("hostPointer", ctypes.c_void_p)]
for gb in (8.6, 17.2):
    n = int(gb * 1e9 / 4)
    t = time.perf_counter()
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    a = Attr()
    r = rt.cudaPointerGetAttributes(ctypes.byref(a), ctypes.c_void_p(h.data_ptr()))
    print(f"{gb} GB: is_pinned={h.is_pinned()} attr rc={r} type={a.type} ({time.perf_counter()-t:.1f} s)")
    del h
