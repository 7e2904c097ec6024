"""Phase breakdown of mpskq_gram_host at the headline shape (pinned vs
pageable K): seconds[] = (encode+simulate, overlap [+ streamed host rows],
-, trailing copy).  Usage: python tools/e2e_breakdown.py [N]"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_09336_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6400
m = 165
lib = N.lib()
X = torch.from_numpy(np.random.default_rng(0).uniform(0, 2, (n, m))).pin_memory()
for label, K in (("pinned", torch.empty((n, n), dtype=torch.float64).pin_memory()),
                 ("pageable", torch.empty((n, n), dtype=torch.float64))):
    secs = np.zeros(4)
    rows = []
    for it in range(6):
        t0 = time.perf_counter()
        N.check(lib.mpskq_gram_host(N.KIND_TRAIN, m, 2, 1, 0.1, 1e-24, 0, 0,
                                    C.cast(X.data_ptr(), C.POINTER(C.c_double)), n, None, 0,
                                    C.cast(K.data_ptr(), C.POINTER(C.c_double)), None,
                                    N.ptr(secs, C.c_double)))
        wall = 1e3 * (time.perf_counter() - t0)
        if it >= 2:
            rows.append([1e3 * secs[0], 1e3 * secs[1], 1e3 * secs[3], wall])
    r = np.mean(rows, axis=0)
    print(f"{label:9s} sim {r[0]:7.2f} ms  overlap {r[1]:7.2f} ms  copy {r[2]:6.2f} ms  host wall {r[3]:7.2f} ms")
