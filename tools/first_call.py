"""First-call latency of the device KNN (module loading etc.), small input."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

t0 = time.perf_counter()
from paper_2408_05459_b200 import _lib, knn  # noqa: E402
_lib.require_device()
torch.cuda.synchronize()
print(f"import + device check {time.perf_counter() - t0:.3f}s")
X = np.abs(np.random.default_rng(0).standard_normal((600, 50)))
for rep in range(3):
    t0 = time.perf_counter()
    ids, sc = knn.knn_search_exact_device(X, 10)
    torch.cuda.synchronize()
    print(f"knn call {rep}: {time.perf_counter() - t0:.3f}s")
Xb = (np.random.default_rng(1).random((600, 80)) < 0.1).astype(np.float64)
for rep in range(2):
    t0 = time.perf_counter()
    ids, sc = knn.knn_search_exact_device(Xb, 10)
    torch.cuda.synchronize()
    print(f"knn binary call {rep}: {time.perf_counter() - t0:.3f}s")
