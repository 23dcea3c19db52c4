import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, ctypes as C
import paper_1710_02812_b200 as H
from paper_1710_02812_b200 import configs, hsvd
w = configs.WORKLOADS[int(sys.argv[1])]
x = configs.generate_torch(w, device="cuda")
xh = x.cpu().pin_memory(); del x; torch.cuda.empty_cache()
ctx = H.Context(0)
cfg = H.MatConfig(gamma=1e-12, row_block_rows=w.d, col_block_cols=w.c, max_rank=w.k)
for it in range(3):
    p, dt, m, n, ld, where, _keep = hsvd._matrix_arg(xh)
    h = C.c_void_p(); cc = cfg._c()
    t0 = time.perf_counter()
    hsvd._check(ctx.lib.hsvd_cu_rank_k_svd(ctx.handle, p, dt, m, n, ld, where, C.byref(cc), C.byref(h)))
    ctx.synchronize(); t1 = time.perf_counter()
    rank = C.c_int64(); ur = C.c_int64(); vr = C.c_int64()
    hsvd._check(ctx.lib.hsvd_cu_result_info(h, C.byref(rank), None, None, C.byref(ur), C.byref(vr), None))
    k = rank.value
    u = np.empty((ur.value, k)); t2 = time.perf_counter()
    hsvd._check(ctx.lib.hsvd_cu_result_u(h, u.ctypes.data)); t3 = time.perf_counter()
    u2 = np.empty((ur.value, k)); u2.fill(0); t4 = time.perf_counter()
    hsvd._check(ctx.lib.hsvd_cu_result_u(h, u2.ctypes.data)); t5 = time.perf_counter()
    v = np.empty((vr.value, k)); hsvd._check(ctx.lib.hsvd_cu_result_v(h, v.ctypes.data)); t6 = time.perf_counter()
    ctx.lib.hsvd_cu_result_free(h)
    print(f"call {1e3*(t1-t0):.1f} ms  u({u.nbytes/1e6:.0f} MB) fresh {1e3*(t3-t2):.1f}  prefaulted {1e3*(t5-t4):.1f} (fill {1e3*(t4-t3):.1f})  v {1e3*(t6-t5):.1f}")
