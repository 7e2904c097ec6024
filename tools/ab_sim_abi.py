"""Simulation device time through the stable C ABI only (mpskq_simulate and the
round-1 entry points), so libraries of different rounds can be A/B-ed with
MPSKQ_LIB on the same box:
    MPSKQ_LIB=... python tools/ab_sim_abi.py m d budget n cap"""
import ctypes as C
import os
import sys

import numpy as np
import torch

m, d, budget, n, cap = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
lib = C.CDLL(os.environ.get("MPSKQ_LIB", "paper_2411_09336_b200/libmpskq.so"))
i64 = C.c_int64
ng, npar = i64(0), i64(0)
lib.mpskq_feature_map_topology(m, 2, d, None, None, None, None, i64(0), C.byref(ng), C.byref(npar))
arr = [np.zeros(ng.value, dtype=np.int32) for _ in range(4)]
P = lambda a: a.ctypes.data_as(C.c_void_p)
lib.mpskq_feature_map_topology(m, 2, d, *(P(a) for a in arr), i64(ng.value), C.byref(ng), C.byref(npar))
nops = i64(0)
lib.mpskq_program_compile(m, i64(ng.value), *(P(a) for a in arr), None, i64(0), C.byref(nops), None, None)
ops = np.zeros((nops.value, 4), dtype=np.int32)
lib.mpskq_program_compile(m, i64(ng.value), *(P(a) for a in arr), P(ops), i64(nops.value), C.byref(nops), None, None)
off = np.zeros(m + 1, dtype=np.int64)
stride = i64(0)
lib.mpskq_batch_layout(m, cap, P(off), C.byref(stride))
dev = torch.device("cuda")
X = torch.from_numpy(np.random.default_rng(0).uniform(0, 2, (n, m))).to(dev)
coef = torch.empty((n, npar.value, 2), dtype=torch.float64, device=dev)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
lib.mpskq_feature_map_coefficients_device(C.c_void_p(X.data_ptr()), i64(n), m, 2, d, C.c_double(0.1),
                                          C.c_void_p(coef.data_ptr()), C.c_void_p(bad.data_ptr()), sp)
ops_d = torch.from_numpy(ops).to(dev)
off_d = torch.from_numpy(off).to(dev)
sites = torch.empty((n, 2 * stride.value), dtype=torch.float64, device=dev)
chi = torch.empty((n, m + 1), dtype=torch.int32, device=dev)
disc = torch.empty(n, dtype=torch.float64, device=dev)
peak = torch.empty(n, dtype=torch.int32, device=dev)
status = torch.zeros(n, dtype=torch.int32, device=dev)
vp = lambda t: C.c_void_p(t.data_ptr())


def run():
    return lib.mpskq_simulate(m, cap, vp(ops_d), i64(nops.value), i64(ng.value), vp(coef), i64(npar.value), i64(n),
                              C.c_double(budget), 0, vp(off_d), stride, vp(sites), vp(chi), vp(disc), vp(peak),
                              vp(status), None, sp)


assert run() == 0
torch.cuda.synchronize()
ts = []
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
print(f"{os.environ.get('MPSKQ_LIB', 'tree')}: m={m} d={d} n={n} cap={cap}: sim {min(ts):.1f} ms, "
      f"status max {int(status.max())}, chi max {int(chi.max())}")
