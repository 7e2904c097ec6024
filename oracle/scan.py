"""Host-pool driver of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Runs oracle/mps_oracle.simulate_row (bitwise the reference's
simulate_dataset → simulate_circuit, kernel.py:128-135 / mps.py:250-257) over
many rows in a process pool so the at-scale parity tests
(tests/test_gpu_scale_parity.py) can compare EVERY GPU state's bond
dimensions with the reference algorithm.  Imported only by tests/ and
tools/parity_scan.py; the product package never imports it.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np


def _row(job):
    idx, x, m, r, d, gamma, budget, keep = job
    from oracle import mps_oracle as O

    st = O.simulate_row(x, m, r, d, gamma, budget)
    return idx, st.bond_dims(), st.discard, (st.sites if keep else None)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_states(X, m: int, r: int, d: int, gamma: float, budget: float, keep=(), processes: int | None = None):
    """(bond dims int32 (n, m+1), accumulated discards (n,), {row: sites}) for
    every row of X, computed by the oracle in a spawn-context pool (safe after
    CUDA initialisation).  Site tensors are returned only for rows in `keep`."""
    keep = set(int(k) for k in keep)
    jobs = [(i, np.asarray(x), m, r, d, gamma, budget, i in keep) for i, x in enumerate(X)]
    procs = processes or host_cores()
    # one BLAS thread per worker: the children import numpy before _row runs,
    # so the setting must be in the environment they are spawned with
    saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    os.environ.update({k: "1" for k in saved})
    try:
        with mp.get_context("spawn").Pool(procs) as pool:
            res = pool.map(_row, jobs, chunksize=max(1, len(jobs) // (8 * procs)))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    chi = np.zeros((len(X), m + 1), dtype=np.int32)
    disc = np.zeros(len(X))
    sites = {}
    for idx, bd, ds, st in res:
        chi[idx] = bd
        disc[idx] = ds
        if st is not None:
            sites[idx] = st
    return chi, disc, sites
