"""Padding model of the chi <= 4 overlap: executed vs
algorithmic complex MACs for 32-ket blocks of the headline states, for the
kernel's rules and alternatives (exact block-max padding, per-site choice of
contraction order).

    python tools/pad_model.py [--rows 6400]

Bond dims come from the oracle (bitwise the reference) in a host pool; the
orderings replicate the library's (ket key sort + greedy chi=4 clustering).
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def key_order(chi):
    n, B = chi.shape
    win = (B + 31) // 32
    keys = np.zeros(n, dtype=np.uint64)
    for b in range(B):
        keys |= (chi[:, b] >= 4).astype(np.uint64) << np.uint64(31 - b // win)
    return np.argsort(keys, kind="stable")


def greedy(chi, order, group=512):
    four = chi >= 4
    out = []
    for g0 in range(0, len(order), group):
        idx = list(order[g0:g0 + group])
        S = four[idx]
        alive = np.ones(len(idx), bool)
        cnt = S.sum(1)
        U = None
        for pos in range(len(idx)):
            cand = np.where(alive)[0]
            if pos % 32 == 0:
                j = cand[np.argmax(cnt[cand])]
                U = S[j].copy()
            else:
                j = cand[np.argmin((S[cand] & ~U).sum(1))]
                U |= S[j]
            alive[j] = False
            out.append(idx[j])
    return np.array(out)


def ratio(chi, order, variant, samples=4000, lanes=32):
    c = chi[order]
    nblk = len(c) // lanes
    blk = c[: nblk * lanes].reshape(nblk, lanes, -1)
    rng = np.random.default_rng(0)
    ex = al = 0.0
    for _ in range(samples):
        a = c[rng.integers(len(c))]
        k = blk[rng.integers(nblk)]
        na, na1 = a[:-1], a[1:]
        bs, br = k[:, :-1], k[:, 1:]
        f = (bs * na * 2 * na1 + bs * 2 * na1 * br).sum()
        Ks, Kr = k.max(0)[:-1], k.max(0)[1:]
        if variant == "kernel":  # kb / br padded to 3 or 4 (block narrow flags), bra exact, ar >= 2
            Ks, Kr = np.where(Ks <= 3, 3, 4), np.where(Kr <= 3, 3, 4)
            e = (na * Ks * 2 * Kr + na * 2 * np.maximum(2, na1) * Kr).sum() * lanes
        elif variant == "block_max":
            e = (na * Ks * 2 * Kr + na * 2 * na1 * Kr).sum() * lanes
        else:  # block max + per-site min of ket-first / bra-first order
            e = np.minimum(na * Ks * 2 * Kr + na * 2 * na1 * Kr, Ks * na * 2 * na1 + Ks * 2 * na1 * Kr).sum() * lanes
        ex += e
        al += f
    return ex / al


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=6400)
    a = ap.parse_args()
    from oracle.scan import oracle_states

    X = np.random.default_rng(0).uniform(0.0, 2.0, (a.rows, 165))
    chi, _, _ = oracle_states(X, 165, 2, 1, 0.1, 1e-24)
    chi = chi.astype(np.int64)
    go = greedy(chi, key_order(chi))
    for v in ("kernel", "block_max", "block_max_best_order"):
        print(f"{v:22s} executed / algorithmic = {ratio(chi, go, v):.3f}")


if __name__ == "__main__":
    main()
