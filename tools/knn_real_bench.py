"""Time the real-valued tensor-core KNN (level 0) on an Amazon2M/Papers100M
shaped attribute matrix: python tools/knn_real_bench.py [n] [d] [K] [check_rows]."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2408_05459_b200 import knn as kn  # noqa: E402
from paper_2408_05459_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2449029
d = int(sys.argv[2]) if len(sys.argv) > 2 else 100
K = int(sys.argv[3]) if len(sys.argv) > 3 else 10
check = int(sys.argv[4]) if len(sys.argv) > 4 else 200
rng = np.random.default_rng(0)
lab = rng.integers(0, 47, n)
X = synth.continuous_attributes(np.random.default_rng(1), lab, 47, d)
Xd = torch.from_numpy(X).cuda()
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids, sc = kn.knn_search_exact_device(Xd, K, integer=0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"iter {it}: {dt * 1e3:.1f} ms  fallback_rows={kn.LAST_STATS.get('fallback_rows')}  "
          f"alg {2 * n * n * d / dt / 1e12:.0f} TFLOP/s (2n^2d)", flush=True)
# spot-check sampled rows against an exact f64 numpy scan
xn = X / np.linalg.norm(X, axis=1)[:, None]
q = rng.choice(n, check, replace=False)
S = xn[q] @ xn.T
S[np.arange(check), q] = -1
got = ids.cpu().numpy()[q]
bad = 0
for r in range(check):
    top = np.lexsort((np.arange(n), -S[r]))[:K]
    if set(top.tolist()) != set(got[r].tolist()):
        kth = S[r][top[-1]]
        diff = set(top.tolist()) ^ set(got[r].tolist())
        if not all(abs(S[r][j] - kth) <= 1e-12 for j in diff):
            bad += 1
print(f"sampled rows checked: {check}, mismatches: {bad}")
