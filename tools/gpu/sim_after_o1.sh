timeout 600 python - <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows
from paper_2411_09336_b200.mps import overlap_matrix
X2 = np.random.default_rng(0).uniform(0, 2, (800, 50)); c2 = P.FeatureMapConfig(50, 2, 2, 0.1)
def sim2(tag):
    for k in range(3):
        b = simulate_rows(X2, c2, 1e-24)
        print(tag, k, 'cap', b.chi_cap, 'dev %.1f ms' % (1e3 * b.seconds), flush=True)
sim2('before')
Xh = np.random.default_rng(0).uniform(0, 2, (64, 8)); ch = P.FeatureMapConfig(8, 2, 1, 0.5)
bh = simulate_rows(Xh, ch, 0.0)
K = overlap_matrix(bh, bh, 'train'); torch.cuda.synchronize()
sim2('after-o1')
b2 = simulate_rows(X2, c2, 1e-24)
K = overlap_matrix(b2, b2, 'train'); torch.cuda.synchronize()
sim2('after-mma12')
PY
