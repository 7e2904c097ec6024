timeout 600 python tools/bench_configs.py config2_m50_d2 2>&1 | cut -c1-200
timeout 600 python tools/bench_configs.py config1_m8_d1 config2_m50_d2 2>&1 | cut -c1-200
timeout 600 python - <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows
for m, d, budget, n in [(8, 1, 0.0, 64), (50, 2, 1e-24, 800)]:
    X = np.random.default_rng(0).uniform(0, 2, (n, m)); cfg = P.FeatureMapConfig(m, 2, d, 0.1 if m > 8 else 0.5)
    for k in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        b = simulate_rows(X, cfg, budget)
        torch.cuda.synchronize(); print(m, k, 'cap', b.chi_cap, 'wall %.1f ms' % (1e3 * (time.perf_counter() - t)), 'dev %.1f ms' % (1e3 * b.seconds))
PY
