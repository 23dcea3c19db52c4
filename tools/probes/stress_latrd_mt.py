"""Concurrent eigensolves from several host threads, one context (stream)
each, to expose cross-stream interactions of the clustered k_latrd."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1710_02812_b200 as H  # noqa: E402

threads = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prog = [0] * threads


def body(r):
    ctx = H.Context(0)
    rng = np.random.default_rng(r)
    n = (300, 700, 384, 1100)[r % 4]
    x = rng.standard_normal((n + 7, n))
    a = x.T @ x
    for i in range(reps):
        H.syevx_topk(a, 20, ctx)
        prog[r] = i + 1


th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(threads)]
for t in th:
    t.start()
t0 = time.time()
while any(t.is_alive() for t in th):
    time.sleep(2)
    print(f"t={time.time() - t0:.0f}s progress={prog}", flush=True)
    if time.time() - t0 > 60:
        print("HUNG", flush=True)
        os._exit(3)
print("ok", prog, flush=True)
